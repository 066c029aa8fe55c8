import sys, time
sys.path.insert(0, ".")
import torch
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate_data
x, spec, m, w = generate_data("C5")
n = x.shape[0]
emu = sys.argv[1] == "1"
cfg = us.Config(memory_cap_entries=max(2 ** 31, n * n + 1), fp64_emulation=emu)
t = torch.from_numpy(x).cuda()
t0 = time.time()
try:
    print("emulation", emu, "u", us.u_statistic(spec, t, config=cfg), "s", time.time() - t0, flush=True)
except Exception as e:
    print("emulation", emu, "FAILED", e, flush=True)
