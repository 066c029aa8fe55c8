"""C5 at n = 65536 with different K-chunk lengths of the emulated GEMM
(Config.oz_max_k): seconds per evaluation, second of two evaluations."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate_data
n = 65536
data, spec, m, _ = generate_data("C5", n)
dX = torch.from_numpy(data).cuda()
for max_k in [int(a) for a in sys.argv[1:]] or [0]:
    cfg = us.Config(memory_cap_entries=max(2 ** 31, n * n + 1), oz_max_k=max_k)
    ts = []
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.time()
        u, st = us.u_statistic(spec, dX, config=cfg, with_stats=True)
        torch.cuda.synchronize(); ts.append(time.time() - t0)
    print(f"oz_max_k={max_k}: {ts[-1]:.2f} s (first {ts[0]:.2f}), u={u!r}, launches={st['kernel_launches']}", flush=True)
