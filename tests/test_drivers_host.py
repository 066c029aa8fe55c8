"""Callers of the path: dcov_squared and motif_count. CPU side:
the reference oracle pinned against independent brute force (subset census,
the O(n^4) dcov sum of acceptance criterion 7) and the engine's argument
validation, which fails before any device work."""
import itertools

import numpy as np
import pytest

import paper_2508_12627_b200 as us
from oracle import ref as REF

# induced patterns (motifs.hpp:33-36): present edges, 1-based
PATTERNS = {
    "r1": (3, [(1, 2), (2, 3)]), "r2": (3, [(1, 2), (1, 3), (2, 3)]),
    "r3": (4, [(1, 2), (1, 3), (1, 4)]), "r4": (4, [(1, 2), (2, 3), (3, 4)]),
    "r5": (4, [(1, 2), (1, 3), (2, 3), (3, 4)]), "r6": (4, [(1, 2), (2, 3), (3, 4), (1, 4)]),
    "r7": (4, [(1, 2), (1, 3), (1, 4), (2, 3), (2, 4)]), "r8": (4, [(1, 2), (1, 3), (1, 4), (2, 3), (2, 4), (3, 4)]),
}
K4 = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
P4 = [(0, 1), (1, 2), (2, 3)]
# test_cli.cpp:328-345
K4_COUNTS = {"r1": 0, "r2": 4, "r3": 0, "r4": 0, "r5": 0, "r6": 0, "r7": 0, "r8": 1}
P4_COUNTS = {"r1": 2, "r2": 0, "r3": 0, "r4": 1, "r5": 0, "r6": 0, "r7": 0, "r8": 0}


def census(n, edges, motif):
    """Vertex subsets whose induced subgraph is isomorphic to the pattern."""
    k, pat = PATTERNS[motif]
    adj = {frozenset(e) for e in map(tuple, edges)}
    want = {frozenset((a - 1, b - 1)) for a, b in pat}
    count = 0
    for sub in itertools.combinations(range(n), k):
        induced = {frozenset((i, j)) for i, j in itertools.combinations(range(k), 2)
                   if frozenset((sub[i], sub[j])) in adj}
        if len(induced) != len(want):
            continue
        if any({frozenset((p[a], p[b])) for a, b in map(tuple, want)} == induced
               for p in itertools.permutations(range(k))):
            count += 1
    return count


def random_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    return [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p]


def dcov_brute(x, y):
    """O(n^4) ordered distinct-index sum (acceptance_main.cpp:353-382), vectorised."""
    d1 = np.sqrt(((x[:, None, :] - x[None, :, :]) ** 2).sum(-1))
    d2 = np.sqrt(((y[:, None, :] - y[None, :, :]) ** 2).sum(-1))
    n = len(x)
    total = 0.0
    for i, j, p, q in itertools.permutations(range(n), 4):
        total += d1[i, j] * (d2[p, q] + d2[i, j] - d2[i, p] - d2[j, q])
    return total / (n * (n - 1) * (n - 2) * (n - 3))


needs_ref = pytest.mark.skipif(not REF.available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("motif", sorted(PATTERNS))
def test_oracle_motif_known_answers(motif):
    assert REF.motif_count(4, K4, motif) == K4_COUNTS[motif]
    assert REF.motif_count(4, P4, motif) == P4_COUNTS[motif]


@needs_ref
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_oracle_motifs_equal_census(seed):
    n = 11
    edges = random_graph(n, 0.4, seed)
    for motif in PATTERNS:
        assert REF.motif_count(n, edges, motif) == census(n, edges, motif)


def test_census_known_answers():
    for motif in PATTERNS:
        assert census(4, K4, motif) == K4_COUNTS[motif]
        assert census(4, P4, motif) == P4_COUNTS[motif]


@needs_ref
@pytest.mark.parametrize("seed", [0, 1])
def test_oracle_dcov_equals_brute_force(seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, size=(9, 2))
    y = 0.5 * x[:, :1] + 0.5 * rng.uniform(-1, 1, size=(9, 1))
    want = dcov_brute(x, y)
    got = REF.dcov_squared(x, y)
    assert abs(got - want) <= 1e-10 * abs(want)


def test_motif_validation_before_device():
    with pytest.raises(us.UStatsError) as e:
        us.motif_count(5, K4, "r9")
    assert e.value.code == "InvalidArgument"
    with pytest.raises(us.UStatsError) as e:
        us.motif_count(5, [(0, 0)], "r2")
    assert e.value.code == "InvalidArgument"
    with pytest.raises(us.UStatsError) as e:
        us.motif_count(3, [(0, 5)], "r2")
    assert e.value.code == "InvalidArgument"
    # fewer vertices than the pattern: zero without any device work (motifs.cpp:59)
    assert us.motif_count(3, [(0, 1), (1, 2)], "r8") == 0
    assert us.motif_count(2, [(0, 1)], "r2") == 0


def test_dcov_validation_before_device():
    x = np.zeros((3, 1))
    with pytest.raises(us.UStatsError) as e:
        us.dcov_squared(x, x)
    assert e.value.code == "SampleTooSmall"
    with pytest.raises(us.UStatsError) as e:
        us.dcov_squared(np.zeros((5, 1)), np.zeros((6, 1)))
    assert e.value.code == "InvalidArgument"
