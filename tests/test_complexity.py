"""complexity_report / chain_signature (complexity.hpp:19-51): the host-side
cost anatomy of a signature. Known answers restated from the reference's
test_complexity.cpp:17-128; random signatures against the reference itself."""
import random

import pytest

import paper_2508_12627_b200 as us
from oracle import ref as REF

# Largest quotient width of the order-m chain, m = 2..8 (test_complexity.cpp:19).
CHAIN_MAX_WIDTH = {2: 1, 3: 1, 4: 2, 5: 2, 6: 2, 7: 2, 8: 3}


@pytest.mark.parametrize("m", range(2, 9))
def test_chain_reports(m):
    r = us.complexity_report(us.chain_signature(m), 10)
    assert r.index_count == m and r.graph_vertices == m and r.graph_edges == m - 1
    assert r.bell_count == us.bell_number(m)
    assert r.sparsified_count == us.bell_number(m - 1)
    assert r.max_quotient_width == CHAIN_MAX_WIDTH[m]
    assert sum(r.count_by_width.values()) == r.sparsified_count
    assert all(0 <= w <= r.max_quotient_width for w in r.count_by_width)
    assert r.treewidth_exact == 1
    assert r.treewidth_lower <= 1 <= r.treewidth_upper


def test_hand_priced_estimates():
    assert us.complexity_report(us.chain_signature(3), 10).flops_estimate == "400"
    r = us.complexity_report(us.chain_signature(4), 10)
    assert r.count_by_width == {1: 4, 2: 1}
    assert r.flops_estimate == "4200"


def test_estimates_past_64_bits_stay_exact():
    r = us.complexity_report(us.chain_signature(4), 10_000_000)
    assert r.flops_estimate == "3000001200000000000000"
    assert r.extent == 10_000_000


def test_disconnected_signature():
    r = us.complexity_report([(1,), (2,)], 10)
    assert (r.bell_count, r.sparsified_count, r.max_quotient_width) == (2, 2, 0)
    assert r.count_by_width == {0: 2}
    assert r.treewidth_exact == 0
    assert r.flops_estimate == "40"


def test_canonicalized_before_pricing():
    a = us.complexity_report(us.chain_signature(4), 7)
    b = us.complexity_report([(0, 1), (1, 2), (2, 3)], 7)
    assert a.flops_estimate == b.flops_estimate and a.count_by_width == b.count_by_width


def test_exactness_bound_and_lifted_quotients():
    r = us.complexity_report(us.chain_signature(6), 10, us.Config(exact_treewidth_bound=4))
    assert r.treewidth_exact is None
    assert r.treewidth_lower >= 1 and r.treewidth_upper >= 1
    assert sum(r.count_by_width.values()) == us.bell_number(5)
    assert r.max_quotient_width == 2


def test_chain_signature_shape_and_errors():
    assert us.chain_signature(2) == [(1, 2)]
    assert us.chain_signature(4) == [(1, 2), (2, 3), (3, 4)]
    with pytest.raises(us.UStatsError):
        us.chain_signature(1)
    with pytest.raises(us.UStatsError):
        us.complexity_report(us.chain_signature(3), 0)


BASELINE_SIGS = {
    "C1": ([(0, 1), (1, 2)], 2000),
    "C2": ([(0, 1), (1, 2), (2, 3), (3, 0)], 8192),
    "C3": ([(0,), (0, 1), (1, 2), (2, 3), (3, 4), (4,)], 16384),
    "C4": ([(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (3, 4), (4, 5)], 1024),
    "C5": ([(0,), (0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6,)], 65536),
}


def _random_signatures(count, seed=7):
    rng = random.Random(seed)
    out = []
    for _ in range(count):
        m = rng.randint(2, 7)
        K = rng.randint(1, 8)
        sig = []
        for _ in range(K):
            order = rng.randint(1, min(3, m))
            sig.append(tuple(rng.sample(range(m), order)))
        out.append(sig)
    return out


@pytest.mark.skipif(not REF.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("sig", [s for s, _ in BASELINE_SIGS.values()] + _random_signatures(40))
def test_matches_reference(sig):
    for extent in (1, 10, 65536):
        mine = us.complexity_report(sig, extent)
        ref = REF.complexity_report(sig, extent)
        for key, val in ref.items():
            assert getattr(mine, key) == val, (key, sig, extent)
