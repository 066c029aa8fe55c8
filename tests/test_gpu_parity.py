"""Parity of the B200 engine with the reference algorithm (CUDA path vs oracle).

Oracles: the numpy restatement (oracle/ustats_np.py) and, when present, the
reference library compiled from its own sources (oracle/_ref). Tolerance is
the north_star's: |U_gpu - U_ref| <= 1e-9 * max_pi |V_pi| (per-term values
compared too).
"""
import itertools

import numpy as np
import pytest

from oracle import ref as REF
from oracle import ustats_np as O

pytestmark = pytest.mark.gpu

TOL = 1e-9


def oracle_terms(factors, sig, m):
    if REF.available():
        rgs, mu, v, _ = REF.u_terms(factors, sig, m)
        return O.combine(mu, v), rgs, mu, v
    u, rows = O.u_statistic(factors, sig, m)
    return u, np.array([r[0] for r in rows]), np.array([r[1] for r in rows]), np.array([r[2] for r in rows])


def check_u(engine, factors, sig, m, config=None):
    u_ref, rgs, mu, v = oracle_terms(factors, sig, m)
    got = engine.u_terms(factors, sig, m, config)
    assert np.array_equal(got.rgs, rgs)
    assert np.array_equal(got.mu, mu)
    scale = max(np.max(np.abs(v)), 1e-300)
    per_term = np.abs(got.v - v) / scale
    assert per_term.max() <= TOL, (per_term, got.v, v)
    assert abs(got.value - u_ref) <= TOL * scale, (got.value, u_ref)
    return got, u_ref


def test_prod2_golden(engine):
    # test_engine.cpp:106-116 / test_smoke.py:43-46
    data = np.array([[1.0], [2.0], [3.0]])
    assert engine.u_statistic("prod2", data) == pytest.approx(22.0, rel=1e-12)
    assert engine.v_statistic("prod2", data) == pytest.approx(36.0, rel=1e-12)


@pytest.mark.parametrize("name,n", [("C1", 64), ("C1", 257), ("C2", 96), ("C2", 130), ("C3", 96),
                                    ("C3", 129), ("C4", 24), ("C4", 33), ("C5", 96), ("C5", 97), ("C5", 130)])
def test_configs_small(engine, name, n):
    from paper_2508_12627_b200.workloads import generate
    factors, sig, m, _ = generate(name, n)
    check_u(engine, factors, sig, m)


@pytest.mark.parametrize("name,n", [("C1", 2000), ("C2", 512), ("C3", 512), ("C4", 64), ("C5", 256)])
def test_configs_medium(engine, name, n):
    from paper_2508_12627_b200.workloads import generate
    factors, sig, m, _ = generate(name, n)
    check_u(engine, factors, sig, m)


@pytest.mark.parametrize("name,n,extra", [("C4", 130, {}), ("C4", 136, {}), ("C5", 200, {}), ("C3", 258, {}),
                                          ("C2", 300, {}), ("C4", 132, dict(shard_rows=True, emulate_world=3)),
                                          ("C5", 520, dict(oz_max_k=128))])
def test_emulated_paths_ragged_small(engine, name, n, extra):
    # the INT8-emulated GEMM, the lazy Khatri-Rao digit split (shared-memory
    # staged, lanes along K), K chunks and row panels at sizes that are not
    # multiples of the 128-row digit panels / 64-byte K tiles (oz_min_dim
    # lowers the emulation threshold), against the reference
    from paper_2508_12627_b200.workloads import generate
    factors, sig, m, _ = generate(name, n)
    got, _ = check_u(engine, factors, sig, m, engine.Config(oz_min_dim=128, memory_cap_entries=2 ** 40, **extra))
    assert got.stats["int8_tensor_ops"] > 0


def random_kernel(m, rng):
    # acceptance_main.cpp:92-125 shape: one or two covering tuples + up to two extras
    slots = list(range(m))
    rng.shuffle(slots)
    cut = int(rng.integers(1, m + 1))
    tuples = [slots[:cut]] + ([slots[cut:]] if cut < m else [])
    for _ in range(int(rng.integers(0, 3))):
        t = [int(rng.integers(0, m))]
        if rng.integers(0, 3) > 0:
            s = int(rng.integers(0, m))
            if s != t[0]:
                t.append(s)
        tuples.append(t)
    return tuples


def test_random_kernels_vs_brute_force(engine):
    # acceptance criterion 1: U == literal sum, m in {2,3,4}, n in [m, 8]
    rng = np.random.default_rng(101)
    for trial in range(60):
        m = int(rng.integers(2, 5))
        n = int(rng.integers(m, 9))
        sig = random_kernel(m, rng)
        factors = [rng.uniform(-1, 1, size=(n,) * len(t)) for t in sig]
        want = O.u_brute_force(factors, sig, m)
        got = engine.u_statistic_tensors(factors, sig, m)
        assert abs(got - want) <= 1e-9 * max(1.0, abs(want)), (trial, sig, got, want)
        unsp = engine.u_statistic_unsparsified_tensors(factors, sig, m)
        assert abs(unsp - want) <= 1e-9 * max(1.0, abs(want)), (trial, sig, unsp, want)


def test_v_statistic_and_restricted(engine):
    rng = np.random.default_rng(404)
    m, n = 4, 6
    sig = [[0, 1], [1, 2], [2, 3], [0, 2]]
    factors = [rng.uniform(-1, 1, size=(n, n)) for _ in sig]
    v = engine.v_statistic_tensors(factors, sig, m)
    want = O.contract(factors, sig)
    assert abs(v - want) <= 1e-12 * max(1, abs(want))
    for p in O.partitions(m):
        got = engine.restricted_v_tensors(factors, sig, p, m)
        want = O.contract(factors, O.induced(sig, p))
        assert abs(got - want) <= 1e-11 * max(1, abs(want)), p


def test_random_notations_vs_numpy(engine):
    # test_einsum.cpp:120-157 / acceptance criterion 2
    rng = np.random.default_rng(2024)
    letters = "abcdefgh"
    for trial in range(80):
        k = int(rng.integers(1, 5))
        n = int(rng.integers(2, 6))
        inputs = [[int(rng.integers(0, 5)) for _ in range(int(rng.integers(1, 4)))] for _ in range(k)]
        present = []
        for t in inputs:
            for i in t:
                if i not in present:
                    present.append(i)
        rng.shuffle(present)
        out = present[: int(rng.integers(0, min(2, len(present)) + 1))]
        tensors = [rng.uniform(-1, 1, size=(n,) * len(t)) for t in inputs]
        got = engine.einsum(tensors, inputs, out)
        spec = ",".join("".join(letters[i] for i in t) for t in inputs) + "->" + "".join(letters[i] for i in out)
        want = np.einsum(spec, *tensors)
        assert np.allclose(got, want, rtol=1e-11, atol=1e-11), (trial, inputs, out)


def test_every_order_same_value(engine):
    # test_einsum.cpp:159-176
    rng = np.random.default_rng(55)
    n = 3
    inputs = [[0, 1, 2], [2, 3], [3, 4], [4, 0]]
    tensors = [rng.uniform(-1, 1, size=(n,) * len(t)) for t in inputs]
    want = np.einsum("abc,cd,de,ea->b", *tensors)
    for perm in itertools.permutations(range(5)):
        got = engine.einsum(tensors, inputs, [1], order=list(perm))
        assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


def test_gemm_shapes_and_transposes(engine):
    # exercises every DMMA loader orientation and ragged tile edges
    rng = np.random.default_rng(7)
    for n in (5, 127, 128, 129, 300):
        a = rng.normal(size=(n, n))
        b = rng.normal(size=(n, n))
        for ins, out, spec in [([[0, 1], [1, 2]], [0, 2], "ij,jk->ik"), ([[1, 0], [1, 2]], [0, 2], "ji,jk->ik"),
                               ([[0, 1], [2, 1]], [0, 2], "ij,kj->ik"), ([[1, 0], [2, 1]], [2, 0], "ji,kj->ki")]:
            got = engine.einsum([a, b], ins, out)
            assert np.allclose(got, np.einsum(spec, a, b), rtol=1e-12, atol=1e-10), (n, spec)


def test_khatri_rao_step(engine):
    # K=3 operands sharing only the eliminated index (generic_step, einsum.cpp:263-301)
    rng = np.random.default_rng(21)
    n = 9
    a, b, c = (rng.uniform(-1, 1, size=(n, n)) for _ in range(3))
    out, tup = engine.eliminate_index([a, b, c], [[0, 1], [0, 2], [0, 3]], 0)
    assert tup == [1, 2, 3]
    assert np.allclose(out, np.einsum("si,sj,sk->ijk", a, b, c), rtol=1e-12)


def test_errors(engine):
    from paper_2508_12627_b200 import UStatsError, Config
    x = np.ones((3, 3))
    with pytest.raises(UStatsError) as e:
        engine.u_statistic_tensors([x, x, x], [[0, 1], [1, 2], [2, 3]], 4)
    assert e.value.code == "SampleTooSmall"
    a = np.ones((10, 10))
    with pytest.raises(UStatsError) as e:
        engine.einsum([a, a], [[0, 1], [1, 2]], [0, 2], config=Config(memory_cap_entries=50))
    assert e.value.code == "MemoryCapExceeded"
    with pytest.raises(UStatsError) as e:
        engine.einsum([a, a], [[0, 1], [1, 2]], [0, 2], order=[0, 1])
    assert e.value.code == "InvalidArgument"


def test_nonfinite_propagates(engine):
    x = np.array([np.nan, 1.0, 2.0])
    assert np.isnan(engine.v_statistic_tensors([x, np.ones(3)], [[0], [1]], 2))


def test_minimum_sample(engine):
    rng = np.random.default_rng(3)
    for m in (2, 3, 4):
        sig = [[i, i + 1] for i in range(m - 1)]
        A = rng.normal(size=(m, m))
        check_u(engine, [A] * (m - 1), sig, m)


def test_deterministic_bits(engine):
    from paper_2508_12627_b200.workloads import generate
    factors, sig, m, _ = generate("C3", 300)
    a = engine.u_statistic_tensors(factors, sig, m)
    b = engine.u_statistic_tensors(factors, sig, m)
    assert a == b


def test_device_resident_inputs(engine):
    import torch
    from paper_2508_12627_b200.workloads import generate
    factors, sig, m, _ = generate("C2", 200)
    host = engine.u_statistic_tensors(factors, sig, m)
    dev = {}
    dfac = []
    for f in factors:
        if id(f) not in dev:
            dev[id(f)] = torch.from_numpy(f).cuda()
        dfac.append(dev[id(f)])
    got = engine.u_statistic_tensors(dfac, sig, m)
    assert got == host


def test_batch_equals_individual(engine):
    from paper_2508_12627_b200.workloads import generate
    probs = []
    for name, n in (("C3", 160),):
        factors, sig, m, _ = generate(name, n)
        probs.append((factors, sig, m))
        # the same chain without its end vector, sharing the matrix object
        probs.append((factors[1:-2], [[i, i + 1] for i in range(m - 2)], m - 1))
    vals = engine.u_statistic_batch(probs)
    for (f, s, m), v in zip(probs, vals):
        want = engine.u_statistic_tensors(f, s, m)
        u_ref, rows = O.u_statistic(f, s, m)
        scale = max(abs(r[2]) for r in rows)
        assert abs(v - want) <= TOL * scale and abs(v - u_ref) <= TOL * scale


def test_hoif_tau_closed_forms(engine):
    # test_kernels.cpp:109-123: tau telescopes to closed forms in U_2..U_4
    rng = np.random.default_rng(44)
    n = 9
    data = rng.normal(size=(n, 4))
    u = {j: engine.u_statistic(f"hoif:{j}:2", data) for j in (2, 3, 4)}
    for j in (2, 3, 4):
        f, s, m = engine.kernel_tensors(f"hoif:{j}:2", data)
        assert abs(u[j] - O.u_brute_force(f, s, m)) <= 1e-11 * max(1, abs(u[j]))
    assert engine.hoif_tau(2, 2, data) == pytest.approx(u[2], rel=1e-12)
    assert engine.hoif_tau(3, 2, data) == pytest.approx(-u[3] / n, rel=1e-12)
    assert engine.hoif_tau(4, 2, data) == pytest.approx(u[2] + u[3] / n + u[4] / (n * (n - 1)), rel=1e-12)
    with pytest.raises(engine.UStatsError) as e:
        engine.hoif_tau(5, 1, rng.normal(size=(4, 3)))
    assert e.value.code == "SampleTooSmall"


@pytest.mark.parametrize("name,n,world", [("C2", 200, 3), ("C3", 130, 4), ("C4", 40, 3), ("C5", 130, 5),
                                          ("C1", 101, 2), ("C5", 300, 8), ("C5", 257, 2), ("C4", 48, 4),
                                          ("C3", 384, 8)])
def test_row_sharding_emulated(engine, name, n, world):
    # the row-sharding plan (shard.cpp) run by `world` virtual ranks on one
    # device, one after the other: row panels of every op, symmetric products
    # as balanced triangle pieces with their transposes stored by the column
    # owner, partial reductions accumulated == the unsharded result
    from paper_2508_12627_b200.workloads import generate
    factors, sig, m, _ = generate(name, n)
    base = engine.u_terms(factors, sig, m)
    cfg = engine.Config(shard_rows=True, emulate_world=world)
    got = engine.u_terms(factors, sig, m, cfg)
    scale = np.max(np.abs(base.v))
    assert np.max(np.abs(got.v - base.v)) <= TOL * scale
    assert abs(got.value - base.value) <= TOL * scale


def test_row_sharding_single_rank_nccl(engine):
    # the real NCCL path at world size 1 (the only size one GPU allows)
    from paper_2508_12627_b200.workloads import generate
    engine.nccl_init(0, 0, 1, engine.nccl_unique_id())
    factors, sig, m, _ = generate("C2", 256)
    base = engine.u_statistic_tensors(factors, sig, m)
    got = engine.u_statistic_tensors(factors, sig, m, engine.Config(shard_rows=True, world_size=1))
    assert got == base


def test_panel_upload_speculation(engine):
    # host matrices >= 2048 upload in row panels overlapped with the first
    # symmetric GEMM; the second call with the same host buffer speculates on
    # symmetry, and a buffer that stopped being symmetric is caught and redone
    from paper_2508_12627_b200.workloads import generate
    factors, sig, m, _ = generate("C2", 2304)
    first = engine.u_terms(factors, sig, m)
    again = engine.u_terms(factors, sig, m)      # speculative path
    assert np.array_equal(first.v, again.v)
    a = factors[0]
    a[5, 7] += 1.0                               # same pointer, now asymmetric
    fresh = engine.u_terms([a.copy()] * 4, sig, m)  # new pointer: probed before planning
    spec = engine.u_terms(factors, sig, m)       # stale cache: mispredicts, recomputes
    scale = np.max(np.abs(fresh.v))
    assert np.max(np.abs(spec.v - fresh.v)) <= TOL * scale
    _, rows = O.u_statistic([a] * 4, sig, m)
    assert abs(spec.value - O.combine([r[1] for r in rows], [r[2] for r in rows])) <= TOL * scale


@pytest.mark.parametrize("name,n", [("C1", 300), ("C2", 256), ("C3", 200), ("C4", 40), ("C5", 160)])
def test_device_tensorization_matches_host(engine, name, n):
    # components tensorized on the GPU from the raw sample == the reference
    # computed from host-tensorized factors (RBF / cosine-feature projection)
    from paper_2508_12627_b200.workloads import generate, generate_data
    data, spec, m, _ = generate_data(name, n)
    factors, sig, _, _ = generate(name, n)
    got, stats = engine.u_statistic(spec, data, config=engine.Config(memory_cap_entries=2 ** 31), with_stats=True)
    u_ref, rows = O.u_statistic(factors, sig, m)
    scale = max(abs(r[2]) for r in rows)
    assert abs(got - u_ref) <= TOL * scale, (got, u_ref)
    assert stats["tensorize_seconds"] > 0
    if REF.available() and name in ("C1", "C2", "C4"):
        u_ref2, _ = REF.u_statistic_data(spec, data)
        assert abs(got - u_ref2) <= TOL * scale


def test_device_tensorization_resident_sample(engine):
    import torch
    from paper_2508_12627_b200.workloads import generate_data
    data, spec, m, _ = generate_data("C2", 300)
    host = engine.u_statistic(spec, data)
    dev = engine.u_statistic(spec, torch.from_numpy(data).cuda())
    assert dev == host
    with pytest.raises(engine.UStatsError) as e:
        engine.u_statistic("rbf:blob3:1", data)
    assert e.value.code == "InvalidArgument"


def test_plan_cache_reexecutes_identically(engine, monkeypatch):
    # a cached program rebinds new inputs of the same structure: bitwise the
    # result of recording afresh; a structural change (asymmetric input) is a
    # different plan
    from paper_2508_12627_b200.workloads import generate
    fa, sig, m, _ = generate("C2", 160)
    rng = np.random.default_rng(3)
    b = rng.random((160, 160))
    b = (b + b.T) / 2
    fb = [b] * len(sig)
    warm = engine.u_terms(fa, sig, m)
    cached = engine.u_terms(fb, sig, m)
    again = engine.u_terms(fa, sig, m)
    monkeypatch.setenv("USTATS_NO_PLAN_CACHE", "1")
    fresh = engine.u_terms(fb, sig, m)
    assert np.array_equal(cached.v, fresh.v) and cached.value == fresh.value
    assert np.array_equal(warm.v, again.v)
    c = rng.random((160, 160))  # not symmetric: another plan
    fc = [c] * len(sig)
    want = engine.u_terms(fc, sig, m)
    monkeypatch.delenv("USTATS_NO_PLAN_CACHE")
    engine.u_terms(fb, sig, m)
    got = engine.u_terms(fc, sig, m)
    assert np.array_equal(got.v, want.v)
    check_u(engine, fc, sig, m)


@pytest.mark.parametrize("name,n", [("C2", 4096), ("C1", 2000)])
def test_data_path_repeatable_at_scale(engine, name, n):
    # the device-tensorized path at a size where the tensorization, the
    # sparsify kernel and the two launch streams overlap: repeated calls are
    # bitwise equal and equal the host-tensor path (whose probe synchronizes)
    from paper_2508_12627_b200.workloads import generate, generate_data
    data, spec, m, _ = generate_data(name, n)
    vals = [engine.u_statistic(spec, data) for _ in range(4)]
    assert all(v == vals[0] for v in vals), vals
    factors, sig, _, _ = generate(name, n)
    ref = engine.u_terms(factors, sig, m)
    scale = np.max(np.abs(ref.v))
    assert abs(vals[0] - ref.value) <= TOL * scale, (vals[0], ref.value)


@pytest.mark.parametrize("name,n,world", [("C2", 2304, 3), ("C3", 2048, 2)])
def test_emulated_gemm_row_sharding(engine, name, n, world):
    # the INT8-emulated GEMM (n >= 2048) over virtual ranks' row panels / pieces == unsharded;
    # both within the north-star tolerance of the DMMA path
    from paper_2508_12627_b200.workloads import generate
    factors, sig, m, _ = generate(name, n)
    base = engine.u_terms(factors, sig, m)
    assert base.stats["int8_tensor_ops"] > 0
    sharded = engine.u_terms(factors, sig, m, engine.Config(shard_rows=True, emulate_world=world))
    exact = engine.u_terms(factors, sig, m, engine.Config(fp64_emulation=False))
    assert exact.stats["int8_tensor_ops"] == 0
    scale = np.max(np.abs(exact.v))
    assert np.max(np.abs(sharded.v - base.v)) <= 1e-12 * scale
    assert np.max(np.abs(base.v - exact.v)) <= TOL * scale


@pytest.mark.parametrize("name,n", [("C5", 22528), ("C5", 21056)])
def test_emulated_gemm_k_chunks(engine, name, n):
    # K = n beyond the exact int32 bound of the digit products (21000): the
    # emulated GEMM runs as K chunks accumulated in FP64 (C5's chain GEMMs
    # have linear consumers only; C2/C3's C^2 consumers stay on DMMA); within
    # the north-star tolerance of the DMMA path, per V-term. n = 21056: a
    # last chunk one 64-wide K step shorter than the first (its own digit layout)
    from paper_2508_12627_b200.workloads import generate
    factors, sig, m, _ = generate(name, n)
    base = engine.u_terms(factors, sig, m)
    assert base.stats["int8_tensor_ops"] > 0
    exact = engine.u_terms(factors, sig, m, engine.Config(fp64_emulation=False))
    assert exact.stats["int8_tensor_ops"] == 0
    scale = np.max(np.abs(exact.v))
    assert np.max(np.abs(base.v - exact.v)) <= TOL * scale
    assert abs(base.value - exact.value) <= TOL * scale


def test_emulated_gemm_k_chunks_row_sharded(engine):
    # the multi-GPU decomposition of C5 (row sharding: each rank its row panel
    # or triangle pieces of every GEMM, digitizing only its operand rows, per K
    # chunk), on virtual ranks: equal to the unsharded K-chunked evaluation
    from paper_2508_12627_b200.workloads import generate
    factors, sig, m, _ = generate("C5", 21056)
    base = engine.u_terms(factors, sig, m)
    sharded = engine.u_terms(factors, sig, m, engine.Config(shard_rows=True, emulate_world=3))
    assert sharded.stats["int8_tensor_ops"] > 0
    scale = np.max(np.abs(base.v))
    assert np.max(np.abs(sharded.v - base.v)) <= 1e-12 * scale


def test_graph_replay_of_repeated_small_evaluations(engine):
    # u_statistic(spec, data) on the same buffers: call 1 records the plan,
    # call 2 captures the whole evaluation (upload, tensorization, kernels,
    # D2H of the terms) as a CUDA graph, later calls replay it. Same kernels in
    # the same order: bit-identical to the plain path; new contents of the same
    # buffer are picked up; what cannot be captured falls back silently.
    import torch
    from paper_2508_12627_b200.workloads import generate, generate_data
    plain = engine.Config(graph_replay=False)
    data, spec, m, _ = generate_data("C1", 600)
    X = torch.from_numpy(data).cuda()
    base = engine.u_statistic(spec, X, config=plain)
    factors, sig, _, _ = generate("C1", 600)
    u_ref, _, _, v = oracle_terms(factors, sig, m)
    assert abs(base - u_ref) <= TOL * np.max(np.abs(v))
    before = engine.graph_replays()
    vals = [engine.u_statistic(spec, X) for _ in range(6)]
    assert all(x == base for x in vals), (vals, base)
    assert engine.graph_replays() - before >= 3
    u, st = engine.u_statistic(spec, X, with_stats=True)
    assert u == base and st["partitions_evaluated"] == len(v)
    # the replayed graph reads the buffer again: new data, new value
    rng = np.random.default_rng(7)
    X.copy_(torch.from_numpy(rng.normal(size=data.shape)))
    torch.cuda.synchronize()
    changed = engine.u_statistic(spec, X)
    assert changed == engine.u_statistic(spec, X, config=plain) and changed != base
    # pinned host sample (H2D inside the graph)
    H = torch.from_numpy(data).pin_memory()
    before = engine.graph_replays()
    assert all(engine.u_statistic(spec, H) == base for _ in range(5))
    assert engine.graph_replays() - before >= 2
    # pageable host memory is not eligible; the projection kernel's host Cholesky cannot be captured
    assert all(engine.u_statistic(spec, data) == base for _ in range(3))
    d3, spec3, _, _ = generate_data("C3", 200)
    X3 = torch.from_numpy(d3).cuda()
    base3 = engine.u_statistic(spec3, X3, config=plain)
    assert all(engine.u_statistic(spec3, X3) == base3 for _ in range(4))
    # a GEMM-bearing plan (two streams joined inside the capture)
    d2, spec2, _, _ = generate_data("C2", 384)
    X2 = torch.from_numpy(d2).cuda()
    base2 = engine.u_statistic(spec2, X2, config=plain)
    before = engine.graph_replays()
    assert all(engine.u_statistic(spec2, X2) == base2 for _ in range(5))
    assert engine.graph_replays() - before >= 2
