"""Small end-to-end runs of every kernel family for compute-sanitizer."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import generate, generate_data

for name, n in (("C1", 130), ("C2", 200), ("C3", 130), ("C4", 36), ("C5", 130)):
    f, sig, m, _ = generate(name, n)
    r = us.u_terms(f, sig, m, us.Config(memory_cap_entries=2 ** 40))
    print(name, n, r.value, flush=True)
    d, spec, m2, _ = generate_data(name, n)
    print(name, "data", us.u_statistic(spec, d, config=us.Config(memory_cap_entries=2 ** 40)), flush=True)
f, sig, m, _ = generate("C2", 129)   # odd n: gather GEMM path
print("C2 odd", us.u_terms(f, sig, m).value)
f, sig, m, _ = generate("C3", 300)   # split-K tail (multi-wave symmetric GEMM)
print("C3 300", us.u_terms(f, sig, m).value)
rng = np.random.default_rng(0)
x, y = rng.normal(size=(90, 2)), rng.normal(size=(90, 3))
print("dcov", us.dcov_squared(x, y))
edges = [(i, j) for i in range(40) for j in range(i + 1, 40) if rng.random() < 0.2]
print("motif", [us.motif_count(40, edges, k) for k in us.MOTIF_IDS])
f4, s4, m4, _ = generate("C4", 30)
print("rows", us.u_terms(f4, s4, m4, us.Config(shard_rows=True, emulate_world=3)).value)
# the INT8-emulated GEMM, lazy Khatri-Rao digit splits and merged-view stream
# kernels at small n (oz_min_dim lowers the emulation threshold), ragged sizes
emu = dict(oz_min_dim=128, memory_cap_entries=2 ** 40)
for name, n in (("C4", 130), ("C4", 136), ("C5", 200), ("C3", 258), ("C2", 300)):
    f, sig, m, _ = generate(name, n)
    r = us.u_terms(f, sig, m, us.Config(**emu))
    print("emulated", name, n, r.value, r.stats["int8_tensor_ops"], flush=True)
    d, spec, m2, _ = generate_data(name, n)
    print("emulated data", name, us.u_statistic(spec, d, config=us.Config(**emu)), flush=True)
f4, s4, m4, _ = generate("C4", 132)
print("emulated rows", us.u_terms(f4, s4, m4, us.Config(shard_rows=True, emulate_world=3, **emu)).value)
f5, s5, m5, _ = generate("C5", 520)
print("emulated k-chunks", us.u_terms(f5, s5, m5, us.Config(oz_max_k=128, **emu)).value)
