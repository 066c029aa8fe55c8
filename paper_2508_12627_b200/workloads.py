"""Seeded synthetic inputs of the five BASELINE.json configurations.

There is no public dataset on this path; every config is a
seeded generator. The same float64 buffers feed the engine and the CPU
reference. Constructions (BASELINE.json "configs"):

  C1  m=3 chain (1,2)(2,3),                  n=2000,  RBF over X~N(0,1)^{n x 5},  seed 0
  C2  m=4 cycle (1,2)(2,3)(3,4)(4,1),        n=8192,  RBF over X~N(0,1)^{n x 10}, seed 1
  C3  m=5 HOIF chain r(1)B..B e(5),          n=16384, B = Z (Z'Z/n)^-1 Z',        seed 2
  C4  m=6 K4(1..4)·(4,5)(5,6),               n=1024,  RBF over X~N(0,1)^{n x 3},  seed 3
  C5  m=7 HOIF chain r(1)B..B e(7),          n=65536, as C3,                      seed 4

Z holds 64 cosine features cos(pi*k*u_c), k=1..16 for each of the 4 uniform
coordinates (k=0 would make Z'Z singular); B is symmetrized ((B+B')/2) so it
is bitwise symmetric. Signatures are 0-based here.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    m: int
    n: int
    seed: int
    signature: tuple
    kind: str  # "rbf" or "hoif"
    dim: int = 0  # RBF input dimension

    def describe(self) -> str:
        return f"{self.name}: m={self.m} n={self.n} sig={list(map(list, self.signature))} seed={self.seed}"


def _chain(m: int):
    return tuple([(0,)] + [(i, i + 1) for i in range(m - 1)] + [(m - 1,)])


K4_TAIL = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (3, 4), (4, 5))

CONFIGS = {
    "C1": Workload("C1", 3, 2000, 0, ((0, 1), (1, 2)), "rbf", 5),
    "C2": Workload("C2", 4, 8192, 1, ((0, 1), (1, 2), (2, 3), (3, 0)), "rbf", 10),
    "C3": Workload("C3", 5, 16384, 2, _chain(5), "hoif"),
    "C4": Workload("C4", 6, 1024, 3, K4_TAIL, "rbf", 3),
    "C5": Workload("C5", 7, 65536, 4, _chain(7), "hoif"),
}


def rbf_matrix(x: np.ndarray, block: int = 2048) -> np.ndarray:
    """A_ij = exp(-||x_i - x_j||^2 / 2); squared distance summed per coordinate
    (bitwise symmetric)."""
    n = x.shape[0]
    out = np.empty((n, n), dtype=np.float64)
    for r0 in range(0, n, block):
        r1 = min(n, r0 + block)
        d = np.zeros((r1 - r0, n))
        for c in range(x.shape[1]):
            diff = x[r0:r1, c, None] - x[None, :, c]
            d += diff * diff
        np.exp(-0.5 * d, out=out[r0:r1])
    return out


def cosine_features(u: np.ndarray, kmax: int = 16) -> np.ndarray:
    cols = [np.cos(np.pi * k * u[:, c]) for c in range(u.shape[1]) for k in range(1, kmax + 1)]
    return np.stack(cols, axis=1)


def projection_matrix(z: np.ndarray) -> np.ndarray:
    n = z.shape[0]
    gram = z.T @ z / n
    chol = np.linalg.cholesky(gram)
    eye = np.eye(gram.shape[0])
    inv_l = np.linalg.solve(chol, eye)
    omega = inv_l.T @ inv_l
    b = (z @ omega) @ z.T
    b += b.T
    b *= 0.5
    return b


def generate(name: str, n: int | None = None):
    """Returns (factors, signature (0-based lists), m, workload). Factors that
    are the same matrix are the same object (aliased)."""
    w = CONFIGS[name]
    n = w.n if n is None else int(n)
    rng = np.random.default_rng(w.seed)
    sig = [list(t) for t in w.signature]
    if w.kind == "rbf":
        x = rng.standard_normal((n, w.dim))
        a = rbf_matrix(x)
        factors = [a for _ in sig]
    else:
        u = rng.uniform(size=(n, 4))
        r = rng.standard_normal(n)
        e = rng.standard_normal(n)
        b = projection_matrix(cosine_features(u))
        factors = [r] + [b] * (w.m - 1) + [e]
    return factors, sig, w.m, w


def input_bytes(factors) -> int:
    seen, total = set(), 0
    for f in factors:
        if id(f) not in seen:
            seen.add(id(f))
            total += f.nbytes
    return total


# Data-level form of each workload: the raw sample and the kernel spec that
# the engine tensorizes on the device (us_u_statistic_data).
SPECS = {"C1": "rbf:chain3:1", "C2": "rbf:cycle4:1", "C3": "proj:5:16", "C4": "rbf:k4tail:1", "C5": "proj:7:16"}


def generate_data(name: str, n: int | None = None):
    """Returns (data n x d, spec, m, workload): the same draws as generate()."""
    w = CONFIGS[name]
    n = w.n if n is None else int(n)
    rng = np.random.default_rng(w.seed)
    if w.kind == "rbf":
        x = rng.standard_normal((n, w.dim))
    else:
        u = rng.uniform(size=(n, 4))
        r = rng.standard_normal(n)
        e = rng.standard_normal(n)
        x = np.concatenate([u, r[:, None], e[:, None]], axis=1)
    return np.ascontiguousarray(x), SPECS[name], w.m, w
