"""One full-size C5 evaluation (m=7 HOIF chain, n=65536, 34.4 GB matrix) on
one B200: host inputs (H2D inside the call), timing and plan statistics."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2508_12627_b200 as us  # noqa: E402
from paper_2508_12627_b200.workloads import generate  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
t0 = time.time()
factors, sig, m, _ = generate("C5", n)
gen = time.time() - t0
import torch  # noqa: E402
pinned = {}
fx = []
for f in factors:
    if id(f) not in pinned:
        pinned[id(f)] = torch.from_numpy(f).pin_memory()
    fx.append(pinned[id(f)])
del factors
cfg = us.Config(memory_cap_entries=2 ** 40)
txt, plan = us.plan_summary(sig, m, n, cfg)
print("plan", json.dumps(plan), flush=True)
from bench import _host_terms  # noqa: E402
us.profile(True, True)
t1 = time.time()
r = _host_terms(us, fx, sig, m, cfg)
wall = time.time() - t1
prof = us.profile(False, True)
out = {"n": n, "u": r.value, "wall_s": wall, "gen_s": gen, "terms": len(r.v), "stats": r.stats, "profile": prof,
       "gemm_tflops": 2 * r.stats["executed_gemm_macs"] / (prof["gemm_ms"] * 1e-3) / 1e12 if prof["gemm_ms"] else None,
       "max_abs_v": float(np.max(np.abs(r.v)))}
print(json.dumps(out), flush=True)
