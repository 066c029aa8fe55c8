"""Pins the oracle before trusting it: the numpy restatement against the
reference's own known answers and against golden fixtures produced by the
reference library (tests/golden/make_golden.py)."""
import hashlib
from pathlib import Path

import numpy as np
import pytest

from oracle import ref as REF
from oracle import ustats_np as O

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_prod2_known_answers():
    # test_engine.cpp:106-116, test_cli.cpp:132-140, test_smoke.py:43-46
    x = np.array([1.0, 2.0, 3.0])
    u, rows = O.u_statistic([x, x], [[0], [1]], 2)
    assert u == 22.0
    assert O.contract([x, x], [[0], [1]]) == 36.0
    assert O.contract([x, x], [[0], [0]]) == 14.0


def test_chain4_counts():
    # test_engine.cpp:202-226: 15 enumerated, 5 evaluated for the chain-4 kernel
    sig = [[0, 1], [1, 2], [2, 3]]
    assert O.bell(4) == 15
    assert len(O.survivors(sig, 4)) == 5


def test_mobius_values():
    # partition.cpp:138-144 hand values
    assert O.mobius((0, 0)) == -1
    assert O.mobius((0, 0, 0)) == 2
    assert O.mobius((0, 0, 0, 0)) == -6
    assert O.mobius((0, 1, 0, 1)) == 1
    assert O.mobius((0, 1, 2, 3)) == 1


def test_oracle_vs_brute_force():
    rng = np.random.default_rng(101)
    for _ in range(20):
        m = int(rng.integers(2, 5))
        n = int(rng.integers(m, 7))
        sig = [[i, i + 1] for i in range(m - 1)] + [[int(rng.integers(0, m))]]
        factors = [rng.uniform(-1, 1, size=(n,) * len(t)) for t in sig]
        u, _ = O.u_statistic(factors, sig, m)
        assert abs(u - O.u_brute_force(factors, sig, m)) <= 1e-10 * max(1, abs(u))


@pytest.mark.parametrize("fixture", sorted(p.name for p in GOLDEN.glob("*.npz")))
def test_oracle_vs_reference_golden(fixture):
    g = np.load(GOLDEN / fixture)
    name, n = fixture.split("_n")
    n = int(n.split(".")[0])
    if n > 2048:
        pytest.skip("large fixture: checked on the GPU only")
    from paper_2508_12627_b200.workloads import generate
    factors, sig, m, _ = generate(name, n)
    hashes, seen = [], set()
    for f in factors:
        if id(f) not in seen:
            seen.add(id(f))
            hashes.append(hashlib.sha256(np.ascontiguousarray(f).tobytes()).hexdigest())
    assert list(g["sha256"]) == hashes, "regenerated inputs differ from the fixture's bytes"
    if (name == "C5" and n > 512) or (name == "C4" and n > 96):
        pytest.skip("numpy restatement too slow at this size on CPU (fixture checked on the GPU)")
    u, rows = O.u_statistic(factors, sig, m)
    v = np.array([r[2] for r in rows])
    assert np.array_equal(np.array([r[0] for r in rows]), g["rgs"])
    assert np.array_equal(np.array([r[1] for r in rows]), g["mu"])
    scale = np.max(np.abs(g["v"]))
    assert np.max(np.abs(v - g["v"])) <= 1e-9 * scale
    assert abs(u - float(g["u"])) <= 1e-9 * scale


@pytest.mark.skipif(not REF.available(), reason="reference library not built")
def test_reference_library_known_answers():
    x = np.array([1.0, 2.0, 3.0])
    assert REF.u_statistic([x, x], [[0], [1]], 2)[0] == 22.0
    assert REF.v_statistic([x, x], [[0], [1]], 2) == 36.0
    assert REF.restricted_v([x, x], [[0], [1]], 2, [0, 0]) == 14.0
    A = np.random.default_rng(7).uniform(-1, 1, size=(7, 7))
    _, st = REF.u_statistic([A, A, A], [[0, 1], [1, 2], [2, 3]], 4, threads=1)
    assert st["partitions_enumerated"] == 15 and st["partitions_evaluated"] == 5 and st["einsum_calls"] == 5


@pytest.mark.skipif(not REF.available(), reason="reference library not built")
def test_reference_matches_restatement_random():
    rng = np.random.default_rng(2025)
    for _ in range(25):
        m = int(rng.integers(2, 5))
        n = int(rng.integers(m, 7))
        slots = list(range(m))
        rng.shuffle(slots)
        sig = [slots[:2], slots[1:]] if m > 2 else [slots]
        factors = [rng.uniform(-1, 1, size=(n,) * len(t)) for t in sig]
        u_ref, _ = REF.u_statistic(factors, sig, m, threads=1)
        u_np, _ = O.u_statistic(factors, sig, m)
        assert abs(u_ref - u_np) <= 1e-10 * max(1, abs(u_ref))
        assert abs(u_ref - REF.u_brute_force(factors, sig, m)) <= 1e-9 * max(1, abs(u_ref))
