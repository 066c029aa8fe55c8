"""Structure of the optimized device program (host only, no GPU).

With sharing / reordering / fusion disabled the recorded program has exactly
the reference executor's GEMM steps (C2 2, C3 7,
C4 3 + 17 K-way, C5 241). With them enabled, the cross-term planner collapses
them (C2's tr(A^4) becomes one symmetric GEMM whose epilogue squares and sums;
C3's seven GEMMs are all B·B)."""
import pytest

import paper_2508_12627_b200 as us
from paper_2508_12627_b200.workloads import CONFIGS

PLAIN = dict(share=False, reorder=False, fuse_epilogues=False, symmetry=False)
CAP = 2 ** 40


def plan(name, **kw):
    w = CONFIGS[name]
    cfg = us.Config(memory_cap_entries=CAP, **kw)
    return us.plan_summary([list(t) for t in w.signature], w.m, w.n, cfg)


@pytest.mark.parametrize("name,gemms", [("C1", 0), ("C2", 2), ("C3", 7), ("C4", 20), ("C5", 241)])
def test_reference_plan_gemm_counts(name, gemms):
    _, tot = plan(name, **PLAIN)
    assert tot["gemms"] == gemms


def test_c2_single_symmetric_fused_gemm():
    text, tot = plan("C2")
    assert tot["gemms"] == 1 and tot["symmetric_gemms"] == 1 and tot["fused_epilogues"] >= 1
    n = CONFIGS["C2"].n
    tiles = n // 128
    assert tot["gemm_macs"] == n ** 3 // (tiles * tiles) * (tiles * (tiles + 1) // 2)
    assert "SYM nostore | epi sum_all pow=2 -> term" in text
    # the two remaining n^2 passes over A (sum A^4, row sums of A^2) share one sweep
    assert "SWEEP" in text and tot["streams"] == 2


def test_sharing_never_increases_work():
    for name in ("C2", "C3", "C4", "C5"):
        _, base = plan(name, **PLAIN)
        _, opt = plan(name)
        assert opt["gemm_macs"] <= base["gemm_macs"]
        assert opt["gemms"] <= base["gemms"]


def test_c3_c5_collapse():
    _, c3 = plan("C3")
    assert c3["gemms"] == 1
    _, c5 = plan("C5")
    assert c5["gemms"] <= 10


def test_plan_respects_memory_cap():
    w = CONFIGS["C5"]
    with pytest.raises(us.UStatsError) as e:
        us.plan_summary([list(t) for t in w.signature], w.m, w.n, us.Config())
    assert e.value.code == "MemoryCapExceeded"


def test_c5_symmetric_products():
    # B, B^2, B^3 = B*B^2, B^4, B D B and its shared transpose: 6 of the 8
    # GEMMs are symmetric (upper tiles only) and the MAC count reflects it
    text, c5 = plan("C5")
    assert c5["gemms"] == 8 and c5["symmetric_gemms"] >= 6
    n = CONFIGS["C5"].n
    assert c5["gemm_macs"] < 8 * n ** 3 * 0.65
    assert text.count(" SYM ") == c5["symmetric_gemms"]


def test_power_and_diagonal_symmetry_rules():
    # chain r B B B e (m = 5 HOIF chain, C3 shape): B*B symmetric; with the
    # symmetric flag off nothing is symmetric
    w = CONFIGS["C3"]
    sig = [list(t) for t in w.signature]
    _, sym = us.plan_summary(sig, w.m, 512, us.Config(memory_cap_entries=CAP), inputs_symmetric=True)
    _, nos = us.plan_summary(sig, w.m, 512, us.Config(memory_cap_entries=CAP, symmetry=False), inputs_symmetric=True)
    assert sym["symmetric_gemms"] >= 1 and nos["symmetric_gemms"] == 0
    assert sym["gemm_macs"] < nos["gemm_macs"]


def test_c2_row_power_sweep():
    text, c2 = plan("C2")
    sweep = [l for l in text.splitlines() if "SWEEP" in l]
    assert len(sweep) == 1
    assert "sum_all pow=4" in sweep[0] and "sum_cols pow=2" in sweep[0]
