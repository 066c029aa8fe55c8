"""C2 row-sharded over W virtual ranks in lockstep on one GPU: total time of
the W slices (a proxy for the per-rank GEMM quantization at W GPUs)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate_data
data, spec, m, _ = generate_data("C2")
dX = torch.from_numpy(data).cuda()
base = us.u_statistic(spec, dX)
for W in (1, 2, 4, 8):
    cfg = us.Config(shard_rows=W > 1, emulate_world=W)
    for _ in range(2):
        u = us.u_statistic(spec, dX, config=cfg)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        u = us.u_statistic(spec, dX, config=cfg)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"W={W} total {dt*1e3:.2f} ms  per-slice {dt*1e3/W:.2f} ms  rel.diff {abs(u-base)/abs(base):.1e}")
