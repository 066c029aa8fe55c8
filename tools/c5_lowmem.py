import sys, time
sys.path.insert(0, ".")
import torch
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate_data
n = 65536
data, spec, m, _ = generate_data("C5", n)
dX = torch.from_numpy(data).cuda()
for hold_gib in (1.0, 2.5):
    hog = torch.empty(int(hold_gib * 2**30), dtype=torch.uint8, device="cuda")
    cfg = us.Config(memory_cap_entries=max(2 ** 31, n * n + 1), exact_treewidth_bound=10 + int(hold_gib))  # distinct plan key per run
    try:
        t0 = time.time()
        u, st = us.u_statistic(spec, dX, config=cfg, with_stats=True)
        torch.cuda.synchronize()
        print(f"held {hold_gib} GiB: {time.time()-t0:.2f} s u={u!r} launches={st['kernel_launches']}", flush=True)
    except Exception as e:
        print(f"held {hold_gib} GiB: {type(e).__name__}: {str(e)[:200]}", flush=True)
    del hog
    torch.cuda.empty_cache()
