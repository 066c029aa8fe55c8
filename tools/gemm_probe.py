"""Times one plain DMMA GEMM (n^3) through the einsum entry point and checks it."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2508_12627_b200 as us  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rng = np.random.default_rng(0)
A = rng.normal(size=(n, n))
B = rng.normal(size=(n, n))
for spec, ins in [("ij,jk", [[0, 1], [1, 2]]), ("ji,jk", [[1, 0], [1, 2]])]:
    for r in range(reps):
        us.profile(True, True)
        out = us.einsum([A, B], ins, [0, 2])
        p = us.profile(False, True)
        print(f"{spec} n={n}: gemm {p['gemm_ms']:.2f} ms -> {2*n**3/p['gemm_ms']/1e9:.2f} TFLOP/s", flush=True)
    ref = np.einsum(spec + "->ik", A, B) if n <= 4096 else None
    if ref is not None:
        print("  max err", np.abs(out - ref).max())
