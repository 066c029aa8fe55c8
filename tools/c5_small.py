"""One C5 evaluation (host tensors) at a given n, for launch lists / ncu."""
import sys
sys.path.insert(0, ".")
import paper_2508_12627_b200 as us  # noqa: E402
from paper_2508_12627_b200.workloads import generate  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 22528
factors, sig, m, _ = generate("C5", n)
r = us.u_terms(factors, sig, m)
print("u", r.value, r.stats.get("int8_tensor_ops"))
