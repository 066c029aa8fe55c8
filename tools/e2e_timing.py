"""Per-call wall time of device-resident vs pinned-host inputs (speculative panel upload)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate
from bench import _host_terms
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
f, sig, m, _ = generate(name)
dev, pin, fx, hx = {}, {}, [], []
for a in f:
    if id(a) not in dev:
        t = torch.from_numpy(a)
        dev[id(a)] = t.cuda(); pin[id(a)] = t.pin_memory()
    fx.append(dev[id(a)]); hx.append(pin[id(a)])
cfg = us.Config()
def run(k, host):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = _host_terms(us, hx, sig, m, cfg) if host else us.u_terms(fx, sig, m, cfg)
        torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    return ts, r
for host in (False, True, False, True):
    ts, r = run(12, host)
    print("host" if host else "dev ", " ".join("%.1f" % t for t in ts), "| U=%r" % r.value)
us.profile(True, True); run(5, True); print("host profile", us.profile(False, True))
us.profile(True, True); run(5, False); print("dev  profile", us.profile(False, True))
