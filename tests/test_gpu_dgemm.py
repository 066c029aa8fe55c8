"""The two FP64 GEMM engines behind the executor (us_dgemm): DMMA (mma.sync
f64) and Ozaki splitting on the INT8 tcgen05 tensor cores, against numpy."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (300, 200, 257), (1000, 130, 2049), (129, 1100, 640)])
def test_ozaki_matches_numpy(engine, m, n, k):
    rng = np.random.default_rng(m + n + k)
    a, b = rng.normal(size=(m, k)), rng.normal(size=(n, k))
    ref = a @ b.T
    got = engine.dgemm(a, b, "ozaki", 7)
    # 7 balanced 8-bit digits: ~2^-54 K max|a| max|b| per entry
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    if k % 2 == 0:  # the TMA-fed DMMA kernel needs 16-byte aligned rows
        dm = engine.dgemm(a, b, "dmma")
        assert np.max(np.abs(dm - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_ozaki_symmetric_is_bitwise_symmetric(engine):
    rng = np.random.default_rng(1)
    a = rng.normal(size=(700, 333))
    c = engine.dgemm(a, a, "ozaki", 7, symmetric=True)
    assert np.array_equal(c, c.T)
    assert np.max(np.abs(c - a @ a.T)) <= 1e-12 * np.max(np.abs(a @ a.T))


def test_ozaki_precision_grows_with_digits(engine):
    rng = np.random.default_rng(2)
    a, b = rng.uniform(0, 1, size=(256, 512)), rng.uniform(0, 1, size=(256, 512))
    ref = a @ b.T
    errs = [np.max(np.abs(engine.dgemm(a, b, "ozaki", s) - ref)) / np.max(ref) for s in (4, 5, 6, 7)]
    assert all(e2 < e1 for e1, e2 in zip(errs, errs[1:]))
    assert errs[-1] < 1e-12


def test_ozaki_wide_dynamic_range_rows(engine):
    # row scaling: rows of very different magnitudes keep their relative accuracy
    rng = np.random.default_rng(3)
    a = rng.normal(size=(256, 256)) * np.logspace(-150, 150, 256)[:, None]
    b = rng.normal(size=(256, 256))
    ref = a @ b.T
    got = engine.dgemm(a, b, "ozaki", 7)
    row_scale = np.max(np.abs(a), axis=1)[:, None] * np.max(np.abs(b)) * 256
    assert np.all(np.abs(got - ref) <= 1e-12 * row_scale)


def test_ozaki_exponents_beyond_the_fast_scaling_range(engine):
    # rows / columns scaled past 2^511 take the out-of-line exponent path of
    # the epilogue; the rest of the tile stays on the branch-free one
    rng = np.random.default_rng(4)
    a = rng.normal(size=(300, 256))
    b = rng.normal(size=(260, 256))
    a[::7] *= 1e200
    b[::11] *= 1e-200
    ref = a @ b.T
    got = engine.dgemm(a, b, "ozaki", 7)
    scale = np.max(np.abs(a), axis=1)[:, None] * np.max(np.abs(b), axis=1)[None, :] * 256
    assert np.all(np.abs(got - ref) <= 1e-12 * scale)
    c = engine.dgemm(a, a, "ozaki", 7, symmetric=True)
    assert np.array_equal(c, c.T)


def test_ozaki_int32_accumulators_at_the_exact_bound(engine):
    # S = 6, K = 26112: just under the int32-exact bound (26176) that splitting
    # the top digit diagonal over two TMEM accumulators allows (21824 before).
    # Every value has the digits (63, 127, 127, 127, 127, 127): all digit
    # products are positive and near the largest possible, so the fullest
    # accumulator (five products on diagonal 4) reaches 98% of 2^31 -- one more
    # product in it, or an unsplit top diagonal (six), would wrap around.
    k = 26112
    x = float(0x3F7F7F7F7F7F) / 2.0 ** 46
    a = np.full((256, k), x)
    b = np.full((384, k), x)
    ref = k * x * x
    got = engine.dgemm(a, b, "ozaki", 6)
    assert got.shape == (256, 384)
    assert np.max(np.abs(got - ref)) <= 1e-11 * ref
    # signs alternate along K in A: the products cancel pairwise and the result is exactly 0
    a2 = a * np.where(np.arange(k) % 2 == 0, 1.0, -1.0)
    assert np.max(np.abs(engine.dgemm(a2, b, "ozaki", 6))) <= 1e-11 * ref
