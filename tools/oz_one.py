"""One emulated GEMM (for ncu): n x n x n, S digits, symmetric or not."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_12627_b200 as us
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
sym = (sys.argv[2] == "sym") if len(sys.argv) > 2 else True
S = int(sys.argv[3]) if len(sys.argv) > 3 else 6
rng = np.random.default_rng(0)
a = rng.uniform(-1, 1, size=(n, n))
b = a if sym else rng.uniform(-1, 1, size=(n, n))
_, ms = us.dgemm(a, b, "ozaki", S, symmetric=sym, with_time=True)
print(f"n={n} sym={sym} S={S}: {ms:.3f} ms")
