"""C2 per-evaluation timing stability (clock ramp / pool warm-up)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import pynvml
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
f, sig, m, _ = generate("C2")
d = torch.from_numpy(f[0]).cuda()
fx = [d] * 4

def run(k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        r = us.u_terms(fx, sig, m)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3

for i in range(12):
    ms = run(10)
    print("batch %2d: %.2f ms  sm %d MHz  pwr %.0f W" % (i, ms, pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                                  pynvml.nvmlDeviceGetPowerUsage(h) / 1000))
