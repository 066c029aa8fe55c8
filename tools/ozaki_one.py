import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
f, sig, m, _ = generate("C2", n)
A = f[0]
for _ in range(2):
    C, ms = us.dgemm(A, A, "ozaki", int(sys.argv[2]) if len(sys.argv) > 2 else 6, symmetric=True, with_time=True)
print(n, f"{ms:.2f} ms")
