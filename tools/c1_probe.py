import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate
f, sig, m, _ = generate("C1")
d = torch.from_numpy(f[0]).cuda()
fx = [d, d]
for i in range(5):
    us.u_terms(fx, sig, m)
ts = []
for i in range(30):
    t0 = time.perf_counter(); r = us.u_terms(fx, sig, m); ts.append(time.perf_counter() - t0)
print("u_terms wall ms: median %.3f min %.3f" % (1e3 * np.median(ts), 1e3 * min(ts)))
print(r.stats)
import cProfile, pstats
cProfile.run("for _ in range(50): us.u_terms(fx, sig, m)", "/tmp/prof")
pstats.Stats("/tmp/prof").sort_stats("cumulative").print_stats(8)
