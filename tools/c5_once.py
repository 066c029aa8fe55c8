"""One C5 evaluation through the binding's public call (device-resident
sample, GPU tensorization): for ncu captures of the C5 kernels."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate_data, CONFIGS
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
data, spec, m, _ = generate_data("C5", n)
cfg = us.Config(memory_cap_entries=max(2 ** 31, n * n + 1))
dX = torch.from_numpy(data).cuda()
t0 = time.time()
u, st = us.u_statistic(spec, dX, config=cfg, with_stats=True)
print("u", u, "wall", time.time() - t0, "launches", st["kernel_launches"], flush=True)
