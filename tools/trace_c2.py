import sys, time, os
sys.path.insert(0, ".")
import torch
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate
from bench import _host_terms
f, sig, m, _ = generate("C2")
pin = torch.from_numpy(f[0]).pin_memory()
print("pinned:", pin.is_pinned())
hx = [pin] * 4
cfg = us.Config()
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = _host_terms(us, hx, sig, m, cfg)
    print("call %d %.2f ms" % (i, (time.perf_counter() - t0) * 1e3), file=sys.stderr, flush=True)
