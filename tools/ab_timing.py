"""Where do per-call outliers come from: host phases vs device wait."""
import os, sys, time, subprocess
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate
f, sig, m, _ = generate("C2")
d = torch.from_numpy(f[0]).cuda()
fx = [d] * 4
os.environ["USTATS_TRACE"] = "1"
print(subprocess.run(["uptime"], capture_output=True, text=True).stdout, flush=True)
print(subprocess.run(["bash", "-c", "ps -eo pcpu,comm --sort=-pcpu | head -8"], capture_output=True, text=True).stdout, flush=True)
for _ in range(3): us.u_terms(fx, sig, m)
for i in range(25):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    us.u_terms(fx, sig, m)
    torch.cuda.synchronize()
    print("call %.2f ms" % ((time.perf_counter() - t0) * 1e3), file=sys.stderr, flush=True)
