"""Host-side cost of one cached C1 evaluation (data API) vs its GPU time."""
import sys, time, os
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate_data
data, spec, m, _ = generate_data("C1")
dX = torch.from_numpy(data).cuda()
for _ in range(20):
    us.u_statistic(spec, dX)
torch.cuda.synchronize()
R = 200
t = time.perf_counter()
for _ in range(R):
    us.u_statistic(spec, dX)
dt = (time.perf_counter() - t) / R
print(f"wall per call {dt*1e6:.1f} us")
os.environ["USTATS_TRACE"] = "1"
us.u_statistic(spec, dX)
