"""dcov_squared and motif_count on the device (SURVEY 8b callers), against
the reference library, independent brute force and closed-form identities."""
import numpy as np
import pytest

from oracle import ref as REF
from test_drivers_host import K4, K4_COUNTS, P4, P4_COUNTS, PATTERNS, census, dcov_brute, random_graph

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not REF.available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("motif", sorted(PATTERNS))
def test_motif_known_answers(engine, motif):
    assert engine.motif_count(4, K4, motif) == K4_COUNTS[motif]
    assert engine.motif_count(4, P4, motif) == P4_COUNTS[motif]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_motifs_equal_census(engine, seed):
    n = 14
    edges = random_graph(n, 0.4, seed)
    for motif in PATTERNS:
        assert engine.motif_count(n, edges, motif) == census(n, edges, motif)


@needs_ref
@pytest.mark.parametrize("n,p,seed", [(30, 0.3, 606), (30, 0.3, 607), (64, 0.25, 3), (90, 0.1, 4)])
def test_motifs_match_reference(engine, n, p, seed):
    # acceptance criterion 6 (random graphs on 30 vertices, all 8 patterns) and larger
    edges = random_graph(n, p, seed)
    for motif in PATTERNS:
        assert engine.motif_count(n, edges, motif) == REF.motif_count(n, edges, motif), motif


def test_motif_identities_large(engine):
    # n = 1200 (n^3 under the 2^31-entry cap): triangles = tr(A^3)/6, induced P3 = sum C(deg,2) - 3 triangles,
    # K4 = sum_i triangles(N(i)) / 4, all exact integers
    n = 1200
    rng = np.random.default_rng(11)
    upper = np.triu(rng.random((n, n)) < 0.03, 1)
    A = (upper | upper.T).astype(np.float64)
    edges = np.argwhere(upper)
    tri = int(round(np.trace(A @ A @ A) / 6))
    deg = A.sum(1)
    wedges = int(round((deg * (deg - 1) / 2).sum()))
    k4 = 0
    for i in range(n):
        nb = np.flatnonzero(A[i])
        S = A[np.ix_(nb, nb)]
        k4 += int(round(np.trace(S @ S @ S) / 6))
    assert engine.motif_count(n, edges, "r2") == tri
    assert engine.motif_count(n, edges, "r1") == wedges - 3 * tri
    assert engine.motif_count(n, edges, "r8") == k4 // 4


def test_motif_empty_graph(engine):
    assert engine.motif_count(50, [], "r2") == 0
    assert engine.motif_count(50, [], "r3") == 0


def _paired(rng, n):
    dx, dy = rng.integers(1, 4, size=2)
    x = rng.uniform(-1, 1, size=(n, dx))
    y = 0.5 * x[:, np.arange(dy) % dx] + 0.5 * rng.uniform(-1, 1, size=(n, dy))
    return x, y


def test_dcov_equals_brute_force(engine):
    rng = np.random.default_rng(5)
    for _ in range(3):
        x, y = _paired(rng, 10)
        want = dcov_brute(x, y)
        assert abs(engine.dcov_squared(x, y) - want) <= 1e-10 * abs(want)


@needs_ref
def test_dcov_criterion_7(engine):
    # acceptance criterion 7: 20 paired samples of 30, relative error <= 1e-10
    rng = np.random.default_rng(707)
    for _ in range(20):
        x, y = _paired(rng, 30)
        want = REF.dcov_squared(x, y)
        assert abs(engine.dcov_squared(x, y) - want) <= 1e-10 * abs(want)


@needs_ref
@pytest.mark.parametrize("n", [257, 1500])
def test_dcov_large_matches_reference(engine, n):
    rng = np.random.default_rng(n)
    x, y = _paired(rng, n)
    want = REF.dcov_squared(x, y)
    got, stats = engine.dcov_squared(x, y, with_stats=True)
    assert abs(got - want) <= 1e-10 * abs(want)
    assert stats["kernel_launches"] >= 3


def test_dcov_device_resident(engine):
    import torch
    rng = np.random.default_rng(9)
    x, y = _paired(rng, 700)
    host = engine.dcov_squared(x, y)
    dev = engine.dcov_squared(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    assert dev == host
