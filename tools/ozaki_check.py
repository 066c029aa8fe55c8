import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2508_12627_b200 as us
rng = np.random.default_rng(0)
for (m, n, k) in [(128, 64, 64), (256, 128, 128), (300, 200, 257)]:
    A = rng.normal(size=(m, k)); B = rng.normal(size=(n, k))
    ref = A @ B.T
    C = us.dgemm(A, B, "ozaki", 7)
    err = np.abs(C - ref).max() / np.abs(ref).max()
    print(m, n, k, "ozaki rel err", err, flush=True)
from paper_2508_12627_b200.workloads import generate
f, sig, m, _ = generate("C2", 2048)
A = f[0]
ref = A @ A.T
for S in (5, 6, 7):
    C, ms = us.dgemm(A, A, "ozaki", S, symmetric=True, with_time=True)
    print("C2-like 2048 S", S, "rel err max", np.abs(C - ref).max() / np.abs(ref).max(), "sym", np.array_equal(C, C.T), ms, "ms")
for n in (4096, 8192):
    f, sig, m, _ = generate("C2", n)
    A = f[0]
    for meth, S, sym in (("dmma", 7, True), ("ozaki", 7, True), ("ozaki", 6, True), ("ozaki", 7, False)):
        C, ms = us.dgemm(A, A, meth, S, symmetric=sym, with_time=True)
        C, ms = us.dgemm(A, A, meth, S, symmetric=sym, with_time=True)
        flops = 2 * n ** 3 * (0.5 if sym else 1.0)
        print(n, meth, S, "sym" if sym else "full", f"{ms:.2f} ms", f"{flops / ms / 1e9:.1f} TFLOP/s-equiv", flush=True)
    if n == 4096:
        ref = A @ A.T
        C = us.dgemm(A, A, "ozaki", 7, symmetric=True)
        print("4096 rel err", np.abs(C - ref).max() / np.abs(ref).max())
