"""NumPy restatement of the reference's exact U-statistic path.

TEST INFRASTRUCTURE ONLY (parity checker; never the product path).

Follows, function by function:
  * PartitionStream::advance        proj/src/partition.cpp:83-97   (lexicographic RGS)
  * mobius_coefficient              proj/src/partition.cpp:138-144
  * cooccurring_pairs / survivors   proj/src/partition.cpp:181-226
  * induced_signature               proj/src/partition.cpp:236-254
  * sparsify                        proj/src/tensor.cpp:54-76
  * lattice_combination/pairwise    proj/src/engine.cpp:25-34, 47-104
  * u_statistic                     proj/src/engine.cpp:173-193
  * u_brute_force                   proj/src/bruteforce.cpp:57-72
Each V-term is contracted with numpy.einsum (a summation-order-free
restatement of einsum.cpp:404-486); parity is therefore tolerance-based
(1e-9 of max|V|, BASELINE.json north_star).

Pinned in tests/test_oracle.py against the reference's golden values
(test_engine.cpp:106-116 prod2 U=22/V=36/14, chain-4 counts 15/5/5,
Bell/Table-1 survivor counts) and against fixtures produced by the
reference library itself (tests/golden/*.npz, made by
tests/golden/make_golden.py from oracle/_ref).
"""
from __future__ import annotations

import itertools
import string

import numpy as np


def partitions(m: int):
    """All set partitions of {0..m-1} as restricted-growth tuples, coarsest first."""
    rgs = [0] * m
    yield tuple(rgs)
    while True:
        prefix = [0] * m
        run = 0
        for i in range(1, m):
            run = max(run, rgs[i - 1])
            prefix[i] = run
        for i in range(m - 1, 0, -1):
            if rgs[i] <= prefix[i]:
                rgs[i] += 1
                for j in range(i + 1, m):
                    rgs[j] = 0
                break
        else:
            return
        yield tuple(rgs)


def bell(m: int) -> int:
    return sum(1 for _ in partitions(m)) if m > 0 else 1


def mobius(rgs) -> int:
    m = len(rgs)
    blocks = max(rgs) + 1
    mu = -1 if (m - blocks) % 2 else 1
    for b in range(blocks):
        size = sum(1 for x in rgs if x == b)
        for k in range(2, size):
            mu *= k
    return mu


def forbidden_pairs(signature):
    pairs = set()
    for t in signature:
        for a in t:
            for b in t:
                if a < b:
                    pairs.add((a, b))
    return sorted(pairs)


def survivors(signature, m: int):
    bad = forbidden_pairs(signature)
    return [p for p in partitions(m) if all(p[a] != p[b] for a, b in bad)]


def induced(signature, rgs):
    return [[rgs[s] for s in t] for t in signature]


def sparsify(t: np.ndarray) -> np.ndarray:
    out = np.array(t, dtype=np.float64, copy=True)
    if out.ndim < 2:
        return out
    n = out.shape[0]
    for idx in itertools.product(range(n), repeat=out.ndim):
        if len(set(idx)) < out.ndim:
            out[idx] = 0.0
    return out if out.ndim > 2 else out


def sparsify_matrix(t: np.ndarray) -> np.ndarray:
    out = np.array(t, dtype=np.float64, copy=True)
    np.fill_diagonal(out, 0.0)
    return out


def contract(tensors, tuples) -> float:
    """Full contraction of tensors over tuples (repeated ids = diagonal reads)."""
    letters = string.ascii_letters
    spec = ",".join("".join(letters[i] for i in t) for t in tuples) + "->"
    return float(np.einsum(spec, *tensors, optimize="greedy"))


def pairwise_sum(terms):
    if len(terms) == 0:
        return 0.0
    if len(terms) <= 4:
        acc = terms[0]
        for x in terms[1:]:
            acc += x
        return acc
    half = len(terms) // 2
    return pairwise_sum(terms[:half]) + pairwise_sum(terms[half:])


def combine(mu, v):
    terms = [float(a) * float(b) for a, b in zip(mu, v)]
    total = 0.0
    for at in range(0, len(terms), 512):
        total += pairwise_sum(terms[at:at + 512])
    return total


def u_statistic(factors, signature, m: int):
    """Returns (U, [(rgs, mu, V)]) for a tensor-backed kernel (0-based signature)."""
    sp = [sparsify_matrix(f) if np.ndim(f) == 2 else (sparsify(f) if np.ndim(f) > 2 else np.asarray(f, float))
          for f in factors]
    rows = []
    for p in survivors(signature, m):
        rows.append((p, mobius(p), contract(sp, induced(signature, p))))
    return combine([r[1] for r in rows], [r[2] for r in rows]), rows


def u_brute_force(factors, signature, m: int) -> float:
    """Literal sum over injective index tuples (bruteforce.cpp:57-72)."""
    n = np.shape(factors[0])[0]
    total = 0.0
    for idx in itertools.permutations(range(n), m):
        prod = 1.0
        for f, t in zip(factors, signature):
            prod *= f[tuple(idx[s] for s in t)]
        total += prod
    return total
