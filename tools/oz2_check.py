"""CTA-pair (2SM) vs single-SM emulated GEMM: accuracy vs numpy and timing.
Run twice: USTATS_OZ_2SM=1 and USTATS_OZ_2SM=0."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_12627_b200 as us

mode = os.environ.get("USTATS_OZ_2SM", "1")
rng = np.random.default_rng(0)
for (m, n, k, sym) in [(300, 200, 257, False), (1000, 130, 2049, False), (129, 1100, 640, False), (700, 700, 333, True),
                       (384, 384, 1024, True), (1280, 1280, 4096, True), (2048, 640, 3000, False)]:
    a = rng.normal(size=(m, k))
    b = a if sym else rng.normal(size=(n, k))
    ref = a @ b.T
    got = us.dgemm(a, b, "ozaki", 7, symmetric=sym)
    err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
    print(f"[{mode}] m={m} n={n} k={k} sym={sym}: rel err {err:.2e} symm={np.array_equal(got, got.T) if sym else '-'}", flush=True)
for (m, k, sym, S) in [(8192, 8192, True, 6), (8192, 8192, False, 6), (16384, 16384, True, 6)]:
    a = rng.uniform(-1, 1, size=(m, k))
    b = a if sym else rng.uniform(-1, 1, size=(m, k))
    us.dgemm(a, b, "ozaki", S, symmetric=sym)
    best = 1e30
    for _ in range(3):
        _, ms = us.dgemm(a, b, "ozaki", S, symmetric=sym, with_time=True)
        best = min(best, ms)
    T = m // 128
    tiles = T * (T + 1) // 2 if sym else T * T
    ops = 2.0 * tiles * 128 * 128 * k * S * (S + 1) // 2
    print(f"[{mode}] {m}^2 x {k} sym={sym} S={S}: {best:.3f} ms  {ops / best / 1e9:.1f} TOPS int8", flush=True)
