"""Python mirror of the reference's binding (proj/python/ustats_py.cpp:68-174)
plus the tensor-level entry points the B200 engine adds.

Names, argument meaning and error behaviour follow ``_ustats``: failures raise
``UStatsError`` whose ``code`` is the reference ErrorCode name.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as N

ERROR_CODES = [
    "InvalidNotation", "InvalidOutput", "ShapeMismatch", "MemoryCapExceeded", "IndexAbsent",
    "TooLargeForExhaustive", "OrderTooLarge", "NotRefinement", "GroundSetMismatch", "VertexAbsent",
    "TooLarge", "OutOfTable", "SampleTooSmall", "TooManyTerms", "NonIntegerResult",
    "ComponentEvaluationError", "InvalidArgument", "CudaError", "CollectiveError",
]

STRATEGIES = {"auto": 0, "min_degree": 1, "min_fill": 2, "exhaustive": 3}


class UStatsError(RuntimeError):
    """Typed engine failure (errors.hpp:10-44); ``code`` is the ErrorCode name."""

    def __init__(self, code: str, message: str):
        super().__init__(message)
        self.code = code


def _check(status: int) -> None:
    if status != 0:
        msg = N.lib().us_last_error().decode(errors="replace")
        code = ERROR_CODES[status - 1] if 0 < status <= len(ERROR_CODES) else "InvalidArgument"
        raise UStatsError(code, msg)


@dataclass
class Config:
    """Config (config.hpp:17-44) + the device section."""

    memory_cap_entries: int = 0       # 0 -> reference default 2**31
    threads: int = 0
    strategy: str = "auto"
    exhaustive_index_bound: int = 0
    exact_treewidth_bound: int = 0
    device: int = -1
    rank: int = 0
    world_size: int = 1
    share: bool = True
    fuse_epilogues: bool = True
    symmetry: bool = True
    reorder: bool = True
    donate_inputs: bool = False  # device inputs sparsified in place (saves one copy)
    shard_rows: bool = False     # multi-GPU: row-shard every op (else V-term sharding)
    serial_launch: bool = False  # one CUDA stream (no GEMM / reduction overlap)
    fp64_emulation: bool = True  # large FP64 GEMMs on the INT8 tensor cores (Ozaki digits); False = DMMA only
    graph_replay: bool = True    # repeated small u_statistic(spec, data) calls replay one captured CUDA graph
    emulate_world: int = 0       # row sharding over virtual ranks on one device (tests)
    memory_budget_bytes: int = 0  # device bytes the memory-bounded schedule may use (0 = free memory)
    oz_slices: int = 0           # emulated-GEMM digit slices (0 = error-bound guard, 4..7 forced)
    oz_max_k: int = 0            # longest emulated K per pass (0 = 21000); longer K runs in chunks
    oz_min_dim: int = 0          # smallest rows / cols / K of an emulated GEMM (0 = 1024; tests lower it)

    def native(self) -> N.UsConfig:
        c = N.UsConfig()
        N.lib().us_config_default(C.byref(c))
        c.memory_cap_entries = self.memory_cap_entries
        c.threads = self.threads
        if self.strategy not in STRATEGIES:
            raise UStatsError("InvalidArgument", f"unknown strategy {self.strategy!r}")
        c.strategy = STRATEGIES[self.strategy]
        c.exhaustive_index_bound = self.exhaustive_index_bound
        c.exact_treewidth_bound = self.exact_treewidth_bound
        c.device = self.device
        c.rank = self.rank
        c.world_size = self.world_size
        c.flags = (1 if self.share else 0) | (2 if self.fuse_epilogues else 0) | \
                  (4 if self.symmetry else 0) | (8 if self.reorder else 0) | (16 if self.donate_inputs else 0) | \
                  (32 if self.shard_rows else 0) | (64 if self.serial_launch else 0) | \
                  (0 if self.fp64_emulation else 128) | (0 if self.graph_replay else 256)
        c.emulate_world = self.emulate_world
        c.memory_budget_bytes = self.memory_budget_bytes
        c.oz_slices = self.oz_slices
        c.oz_max_k = self.oz_max_k
        c.oz_min_dim = self.oz_min_dim
        return c


@dataclass
class UTerms:
    """Per-survivor view of one U evaluation (engine.cpp:67-73)."""

    value: float
    rgs: np.ndarray      # (T, m) int32
    mu: np.ndarray       # (T,) int64
    v: np.ndarray        # (T,) float64 (0 where another rank owns the term)
    owner: np.ndarray    # (T,) int32
    stats: dict = field(default_factory=dict)


# ----------------------------------------------------------------- encoding
def _signature(signature: Sequence[Sequence[int]]):
    lens = [len(t) for t in signature]
    idx = [int(s) for t in signature for s in t]
    L = (N.i32 * max(len(lens), 1))(*lens)
    I = (N.i32 * max(len(idx), 1))(*idx)
    return len(lens), L, I


class _Factors:
    """Keeps the factor buffers alive and exposes a void* array for the ABI.

    Accepts numpy arrays (host) or CUDA tensors exposing ``data_ptr()``
    (device; float64, contiguous). Identical objects stay aliased so the
    engine uploads them once.
    """

    def __init__(self, factors, n: int | None = None):
        self.keep = []
        ptrs = []
        on_device = None
        seen: dict[int, int] = {}
        for f in factors:
            dev = hasattr(f, "data_ptr") and getattr(f, "is_cuda", False)
            if on_device is None:
                on_device = dev
            elif on_device != dev:
                raise UStatsError("InvalidArgument", "factors must all be host arrays or all device tensors")
            if dev:
                if str(f.dtype) != "torch.float64" or not f.is_contiguous():
                    raise UStatsError("InvalidArgument", "device factors must be contiguous float64")
                self.keep.append(f)
                ptrs.append(f.data_ptr())
            else:
                key = id(f)
                if key in seen:
                    ptrs.append(ptrs[seen[key]])
                    continue
                a = np.ascontiguousarray(f, dtype=np.float64)
                self.keep.append(a)
                seen[key] = len(ptrs)
                ptrs.append(a.ctypes.data)
        self.on_device = 1 if on_device else 0
        self.ptrs = (C.c_void_p * max(len(ptrs), 1))(*ptrs)
        if n is None:
            shapes = [getattr(f, "shape", ()) for f in factors]
            n = next((int(s[0]) for s in shapes if len(s) > 0), 1)
        self.n = n


def _cfg(config: Config | None) -> N.UsConfig:
    return (config or Config()).native()


# ------------------------------------------------------- statistic (tensors)
def u_statistic_tensors(factors, signature, m: int | None = None, config: Config | None = None,
                        with_stats: bool = False):
    """U-statistic of a tensor-backed kernel (engine.cpp:173-193 after tensorize).

    ``factors[k]`` is component k over [0,n)^len(signature[k]) (unsparsified),
    ``signature`` 0-based slots."""
    m = m if m is not None else 1 + max(s for t in signature for s in t)
    K, L, I = _signature(signature)
    fx = _Factors(factors)
    out = N.f64()
    st = N.UsStats()
    cfg = _cfg(config)
    _check(N.lib().us_u_statistic(m, K, L, I, fx.ptrs, fx.n, fx.on_device, C.byref(cfg), C.byref(out),
                                   C.byref(st)))
    return (out.value, st.as_dict()) if with_stats else out.value


def u_terms(factors, signature, m: int | None = None, config: Config | None = None) -> UTerms:
    m = m if m is not None else 1 + max(s for t in signature for s in t)
    K, L, I = _signature(signature)
    fx = _Factors(factors)
    cap = int(bell_number(m))
    rgs = np.zeros((cap, m), dtype=np.int32)
    mu = np.zeros(cap, dtype=np.int64)
    v = np.zeros(cap, dtype=np.float64)
    owner = np.zeros(cap, dtype=np.int32)
    count = N.i32()
    u = N.f64()
    st = N.UsStats()
    cfg = _cfg(config)
    _check(N.lib().us_u_terms(m, K, L, I, fx.ptrs, fx.n, fx.on_device, C.byref(cfg), cap, C.byref(count),
                              rgs.ctypes.data_as(C.POINTER(N.i32)), mu.ctypes.data_as(C.POINTER(N.i64)),
                              v.ctypes.data_as(C.POINTER(N.f64)), owner.ctypes.data_as(C.POINTER(N.i32)),
                              C.byref(u), C.byref(st)))
    T = count.value
    return UTerms(u.value, rgs[:T].copy(), mu[:T].copy(), v[:T].copy(), owner[:T].copy(), st.as_dict())


def u_statistic_batch(problems, config: Config | None = None, with_stats: bool = False):
    """Several U-statistics ``[(factors, signature, m), ...]`` over one extent,
    evaluated as one device program (shared uploads and sub-contractions)."""
    ms, Ks, lens, idx, allf = [], [], [], [], []
    for factors, sig, m in problems:
        ms.append(int(m))
        Ks.append(len(sig))
        for t in sig:
            lens.append(len(t))
            idx.extend(int(s) for s in t)
        allf.extend(factors)
    fx = _Factors(allf)
    S = len(ms)
    out = (N.f64 * S)()
    st = N.UsStats()
    cfg = _cfg(config)
    _check(N.lib().us_u_statistic_batch(S, (N.i32 * S)(*ms), (N.i32 * S)(*Ks), (N.i32 * len(lens))(*lens),
                                        (N.i32 * max(len(idx), 1))(*idx), fx.ptrs, fx.n, fx.on_device,
                                        C.byref(cfg), out, C.byref(st)))
    vals = [out[i] for i in range(S)]
    return (vals, st.as_dict()) if with_stats else vals


def hoif_tau(m: int, k: int, data, config: Config | None = None, with_stats: bool = False):
    """hoif_tau (hoif.cpp:74-100) with phi = truncation_phi(k) on a sample of
    rows [A, Y, Z...] (host array or CUDA tensor): the component matrices are
    tensorized on the GPU, every chain order 2..m runs in ONE program (the
    reference makes m - 1 separate u_statistic calls) and the combination
    accumulates in long double, as the reference does (us_hoif_tau)."""
    p, n, d, on_device, keep = _sample_arg(data, "data")
    out = N.f64()
    st = N.UsStats()
    _check(N.lib().us_hoif_tau(m, k, C.c_void_p(p), n, d, on_device, C.byref((config or Config()).native()),
                               C.byref(out), C.byref(st)))
    del keep
    return (out.value, st.as_dict()) if with_stats else out.value


def u_statistic_unsparsified_tensors(factors, signature, m: int | None = None, config: Config | None = None):
    m = m if m is not None else 1 + max(s for t in signature for s in t)
    K, L, I = _signature(signature)
    fx = _Factors(factors)
    out = N.f64()
    cfg = _cfg(config)
    _check(N.lib().us_u_statistic_unsparsified(m, K, L, I, fx.ptrs, fx.n, fx.on_device, C.byref(cfg),
                                               C.byref(out), None))
    return out.value


def v_statistic_tensors(factors, signature, m: int | None = None, config: Config | None = None):
    m = m if m is not None else 1 + max(s for t in signature for s in t)
    K, L, I = _signature(signature)
    fx = _Factors(factors)
    out = N.f64()
    cfg = _cfg(config)
    _check(N.lib().us_v_statistic(m, K, L, I, fx.ptrs, fx.n, C.byref(cfg), C.byref(out), None))
    return out.value


def restricted_v_tensors(factors, signature, rgs, m: int | None = None, config: Config | None = None):
    m = m if m is not None else len(rgs)
    K, L, I = _signature(signature)
    fx = _Factors(factors)
    R = (N.i32 * m)(*[int(x) for x in rgs])
    out = N.f64()
    cfg = _cfg(config)
    _check(N.lib().us_restricted_v(m, K, L, I, fx.ptrs, fx.n, R, C.byref(cfg), C.byref(out), None))
    return out.value


def combine_terms(mu, v) -> float:
    """The reference combination (engine.cpp:47-104) of per-term values."""
    mu = np.ascontiguousarray(mu, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    return N.lib().us_combine_terms(len(mu), mu.ctypes.data_as(C.POINTER(N.i64)),
                                    v.ctypes.data_as(C.POINTER(N.f64)))


# ------------------------------------------------------------------- einsum
def einsum(tensors, inputs, output=(), threads: int = 0, order=None, config: Config | None = None,
           with_stats: bool = False):
    """``_ustats.einsum`` (ustats_py.cpp:73-90): contract tensors over index tuples."""
    arrays = [np.ascontiguousarray(t, dtype=np.float64) for t in tensors]
    if len(arrays) != len(inputs):
        raise UStatsError("ShapeMismatch", f"notation expects {len(inputs)} tensors, got {len(arrays)}")
    n = 1
    for a in arrays:
        if a.ndim:
            n = a.shape[0]
            break
    for a in arrays:
        if any(d != n for d in a.shape):
            raise UStatsError("ShapeMismatch", "tensor axes must share one extent")
    for a, t in zip(arrays, inputs):
        if a.ndim != len(t):
            raise UStatsError("ShapeMismatch", "tensor order does not match its tuple")
    K, L, I = _signature(inputs)
    ptrs = (C.c_void_p * max(K, 1))(*[a.ctypes.data for a in arrays])
    out_t = [int(x) for x in output]
    O = (N.i32 * max(len(out_t), 1))(*out_t)
    ordp, ordn = None, 0
    if order is not None:
        ordn = len(order)
        ordp = (N.i32 * max(ordn, 1))(*[int(x) for x in order])
    res = np.zeros((n,) * len(out_t), dtype=np.float64)
    madds, peak, steps = N.u64(), N.u64(), N.i32()
    cfg = (config or Config(threads=threads)).native()
    _check(N.lib().us_einsum(K, L, I, ptrs, n, len(out_t), O, ordp, ordn, C.byref(cfg),
                             res.ctypes.data_as(C.POINTER(N.f64)), C.byref(madds), C.byref(peak),
                             C.byref(steps)))
    if with_stats:
        return res, {"multiply_adds": madds.value, "peak_intermediate_entries": peak.value,
                     "steps": steps.value}
    return res


def eliminate_index(tensors, tuples, index: int, config: Config | None = None):
    arrays = [np.ascontiguousarray(t, dtype=np.float64) for t in tensors]
    n = arrays[0].shape[0] if arrays and arrays[0].ndim else 1
    K, L, I = _signature(tuples)
    ptrs = (C.c_void_p * max(K, 1))(*[a.ctypes.data for a in arrays])
    ids = sorted({s for t in tuples for s in t})
    cap = n ** max(len(ids) - 1, 0)
    out = np.zeros(cap, dtype=np.float64)
    tup = (N.i32 * max(len(ids), 1))()
    tl = N.i32()
    cfg = _cfg(config)
    _check(N.lib().us_eliminate_index(K, L, I, ptrs, n, index, C.byref(cfg),
                                      out.ctypes.data_as(C.POINTER(N.f64)), cap, tup, C.byref(tl)))
    t = [tup[i] for i in range(tl.value)]
    return out[: n ** len(t)].reshape((n,) * len(t)), t


# ------------------------------------------------------- kernel specs (data)
def kernel_tensors(kernel: str, data):
    """Tensorizes a built-in kernel spec of the binding (ustats_py.cpp:45-57):
    ``prod2`` or ``hoif:<j>:<k>`` (hoif.cpp:50-72). Returns (factors, 0-based signature, m)."""
    x = np.asarray(data, dtype=np.float64)
    if x.ndim != 2:
        raise UStatsError("InvalidArgument", "data must be a 2-D array (rows = observations)")
    if kernel == "prod2":
        if x.shape[1] < 1:
            raise UStatsError("InvalidArgument", "prod2 needs at least one coordinate")
        v = np.ascontiguousarray(x[:, 0])
        return [v, v], [[0], [1]], 2
    if kernel.startswith("hoif:"):
        try:
            _, j, k = kernel.split(":")
            j, k = int(j), int(k)
        except ValueError as e:
            raise UStatsError("InvalidArgument", "expected hoif:<j>:<k>") from e
        if j < 2:
            raise UStatsError("InvalidArgument", "sequential kernel needs order >= 2")
        if k < 1:
            raise UStatsError("InvalidArgument", "basis size must be >= 1")
        if x.shape[1] < 2 + k:
            raise UStatsError("InvalidArgument", "covariate block shorter than the basis")
        a, y, phi = x[:, 0], x[:, 1], x[:, 2:2 + k]
        gram = np.zeros((x.shape[0], x.shape[0]))
        for c in range(k):  # dot accumulated in coordinate order (hoif.cpp:13-19)
            gram += phi[:, c, None] * phi[None, :, c]
        middle = np.ascontiguousarray((a[:, None] * gram) * a[None, :])
        last = np.ascontiguousarray((a[:, None] * gram) * y[None, :])
        factors = [middle] * (j - 2) + [last]
        sig = [[i, i + 1] for i in range(j - 1)]
        return factors, sig, j
    raise UStatsError("InvalidArgument", f"unknown kernel spec '{kernel}' (prod2 | hoif:<j>:<k>)")


def u_statistic(kernel: str, data, threads: int = 0, config: Config | None = None, with_stats: bool = False):
    """``_ustats.u_statistic`` (ustats_py.cpp:92-101): the kernel's components
    are tensorized on the GPU from ``data`` (n x d; a numpy array, or a CUDA
    float64 tensor already resident in HBM). Specs: prod2 | hoif:<j>:<k> |
    rbf:<shape>:<h> | proj:<m>:<kmax> (us_u_statistic_data)."""
    if hasattr(data, "data_ptr"):  # torch tensor: CUDA (resident) or CPU (e.g. pinned)
        if str(data.dtype) != "torch.float64" or not data.is_contiguous() or data.dim() != 2:
            raise UStatsError("InvalidArgument", "tensor data must be a contiguous 2-D float64 tensor")
        on_dev = 1 if getattr(data, "is_cuda", False) else 0
        ptr, n, d, keep = data.data_ptr(), data.shape[0], data.shape[1], data
    else:
        x = np.ascontiguousarray(data, dtype=np.float64)
        if x.ndim == 1:
            x = x.reshape(-1, 1)
        if x.ndim != 2:
            raise UStatsError("InvalidArgument", "data must be a 2-D array (rows = observations)")
        ptr, n, d, on_dev, keep = x.ctypes.data, x.shape[0], x.shape[1], 0, x
    out = N.f64()
    st = N.UsStats()
    cfg = (config or Config(threads=threads)).native()
    _check(N.lib().us_u_statistic_data(kernel.encode(), C.c_void_p(ptr), n, d, on_dev, C.byref(cfg),
                                       C.byref(out), C.byref(st)))
    del keep
    return (out.value, st.as_dict()) if with_stats else out.value


def _sample_arg(data, label):
    """(ptr, n, d, on_device, keepalive) of an n x d float64 sample."""
    if hasattr(data, "data_ptr"):
        if str(data.dtype) != "torch.float64" or not data.is_contiguous() or data.dim() not in (1, 2):
            raise UStatsError("InvalidArgument", f"{label} must be a contiguous float64 tensor")
        d = data.shape[1] if data.dim() == 2 else 1
        return data.data_ptr(), data.shape[0], d, 1 if getattr(data, "is_cuda", False) else 0, data
    x = np.ascontiguousarray(data, dtype=np.float64)
    if x.ndim == 1:
        x = x.reshape(-1, 1)
    if x.ndim != 2:
        raise UStatsError("InvalidArgument", f"{label} must be a 2-D array (rows = observations)")
    return x.ctypes.data, x.shape[0], x.shape[1], 0, x


def dcov_squared(x, y, config: Config | None = None, with_stats: bool = False):
    """``dcov_squared`` (dcov.hpp:22-23): unbiased squared distance covariance
    of paired samples (rows = observations), from four U-statistics over the
    Euclidean distance matrices, built and evaluated on the GPU."""
    px, nx, dx, ox, kx = _sample_arg(x, "x")
    py, ny, dy, oy, ky = _sample_arg(y, "y")
    if nx != ny:
        raise UStatsError("InvalidArgument", "paired samples must have equal sizes")
    if ox != oy:
        raise UStatsError("InvalidArgument", "x and y must both be host or both be device arrays")
    out = N.f64()
    st = N.UsStats()
    _check(N.lib().us_dcov_squared(C.c_void_p(px), dx, C.c_void_p(py), dy, nx, ox,
                                   C.byref((config or Config()).native()), C.byref(out), C.byref(st)))
    del kx, ky
    return (out.value, st.as_dict()) if with_stats else out.value


MOTIF_IDS = ("r1", "r2", "r3", "r4", "r5", "r6", "r7", "r8")


def motif_count(n: int, edges, motif_id: str, config: Config | None = None, with_stats: bool = False):
    """``motif_count`` (motifs.hpp:47-48): induced copies of motif r1..r8 in the
    graph on vertices 0..n-1 with the given (u, v) edges."""
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    out = N.i64()
    st = N.UsStats()
    _check(N.lib().us_motif_count(int(n), e.shape[0], e.ctypes.data_as(C.POINTER(N.i32)), motif_id.encode(),
                                  C.byref((config or Config()).native()), C.byref(out), C.byref(st)))
    return (out.value, st.as_dict()) if with_stats else out.value


def v_statistic(kernel: str, data, threads: int = 0, config: Config | None = None):
    """``_ustats.v_statistic`` (ustats_py.cpp:104-113)."""
    factors, sig, m = kernel_tensors(kernel, data)
    return v_statistic_tensors(factors, sig, m, config or Config(threads=threads))


# ------------------------------------------------------------ host helpers
def bell_number(m: int) -> int:
    if m < 0 or m > 15:
        raise UStatsError("InvalidArgument", "Bell numbers supported for 0 <= m <= 15")
    return int(N.lib().us_bell_number(m))


def survivors(signature, m: int):
    """Sparsification survivors in enumeration order: (rgs (T,m), mu (T,), enumerated)."""
    K, L, I = _signature(signature)
    cap = 1024
    while True:
        rgs = np.zeros((cap, max(m, 1)), dtype=np.int32)
        mu = np.zeros(cap, dtype=np.int64)
        count, en = N.i32(), N.u64()
        st = N.lib().us_survivors(m, K, L, I, cap, C.byref(count), rgs.ctypes.data_as(C.POINTER(N.i32)),
                                  mu.ctypes.data_as(C.POINTER(N.i64)), C.byref(en))
        if st == 1 + ERROR_CODES.index("TooManyTerms") and count.value > cap:
            cap = count.value
            continue
        _check(st)
        return rgs[: count.value].copy(), mu[: count.value].copy(), en.value


def plan_terms(signature, m: int, n: int, world_size: int):
    """Term-sharding plan: (owner (T,), cost (T,)) for the sparsified lattice."""
    K, L, I = _signature(signature)
    cap = bell_number(m)
    owner = np.zeros(cap, dtype=np.int32)
    cost = np.zeros(cap)
    cnt = N.i32()
    _check(N.lib().us_plan_terms(m, K, L, I, n, world_size, cap, C.byref(cnt),
                                 owner.ctypes.data_as(C.POINTER(N.i32)), cost.ctypes.data_as(C.POINTER(N.f64))))
    return owner[: cnt.value].copy(), cost[: cnt.value].copy()


def plan_summary(signature, m: int, n: int, config: Config | None = None, inputs_symmetric: bool = True):
    """Host-only view of the optimized device program: (text, totals dict)."""
    K, L, I = _signature(signature)
    cap = 1 << 22
    buf = C.create_string_buffer(cap)
    tot = (N.u64 * 7)()
    cfg = _cfg(config)
    _check(N.lib().us_plan_summary(m, K, L, I, n, C.byref(cfg), 1 if inputs_symmetric else 0, buf, cap, tot))
    names = ["gemms", "gemm_macs", "streams", "stream_entries", "fused_epilogues", "symmetric_gemms",
             "peak_entries"]
    return buf.value.decode(), dict(zip(names, list(tot)))


def optimize_order(inputs, strategy: str = "auto"):
    K, L, I = _signature(inputs)
    ids = len({s for t in inputs for s in t})
    out = (N.i32 * max(ids, 1))()
    cnt, w = N.i32(), N.i32()
    _check(N.lib().us_optimize_order(K, L, I, STRATEGIES[strategy], out, C.byref(cnt), C.byref(w)))
    return [out[i] for i in range(cnt.value)], w.value


def treewidth(n: int, edges):
    """``_ustats.treewidth`` (ustats_py.cpp:141-150)."""
    flat = [int(v) for e in edges for v in e]
    E = (N.i32 * max(len(flat), 1))(*flat)
    order = (N.i32 * max(n, 1))()
    w = N.i32()
    _check(N.lib().us_treewidth(n, len(edges), E, C.byref(w), order))
    return w.value, [order[i] for i in range(n)]


@dataclass
class ComplexityReport:
    """``ustats::ComplexityReport`` (complexity.hpp:19-44)."""
    index_count: int
    extent: int
    graph_vertices: int
    graph_edges: int
    treewidth_lower: int
    treewidth_upper: int
    treewidth_exact: int | None
    bell_count: int
    sparsified_count: int
    count_by_width: dict
    max_quotient_width: int
    flops_estimate: str


def complexity_report(signature, extent: int, config: Config | None = None) -> ComplexityReport:
    """``complexity_report`` (complexity.hpp:46-47): lattice sizes, the
    survivors' exact quotient-treewidth histogram and the exact FLOP estimate.
    Tuples may be 0- or 1-based."""
    K, L, I = _signature(signature)
    out = N.UsComplexity()
    buf = C.create_string_buffer(512)
    _check(N.lib().us_complexity_report(K, L, I, int(extent), C.byref(_cfg(config)), C.byref(out), buf, 512))
    return ComplexityReport(
        index_count=out.index_count, extent=out.extent, graph_vertices=out.graph_vertices,
        graph_edges=out.graph_edges, treewidth_lower=out.treewidth_lower, treewidth_upper=out.treewidth_upper,
        treewidth_exact=None if out.treewidth_exact < 0 else out.treewidth_exact,
        bell_count=out.bell_count, sparsified_count=out.sparsified_count,
        count_by_width={w: int(c) for w, c in enumerate(out.count_by_width) if c},
        max_quotient_width=out.max_quotient_width, flops_estimate=buf.value.decode())


def chain_signature(m: int):
    """``chain_signature`` (complexity.hpp:51): ((1,2),...,(m-1,m)), 1-based."""
    if m < 2:
        raise UStatsError("InvalidArgument", "chain signature needs order >= 2")
    return [(i, i + 1) for i in range(1, m)]


def dgemm(a, b, method: str = "ozaki", slices: int = 7, symmetric: bool = False, with_time: bool = False):
    """C = A B^T in FP64 on the device: method "dmma" (mma.sync f64) or
    "ozaki" (balanced 8-bit digit splitting on the INT8 tcgen05 tensor cores)."""
    A = np.ascontiguousarray(a, dtype=np.float64)
    B = np.ascontiguousarray(b, dtype=np.float64)
    if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[1]:
        raise UStatsError("InvalidArgument", "dgemm needs A (m x k) and B (n x k)")
    Cm = np.empty((A.shape[0], B.shape[0]))
    ms = N.f64()
    _check(N.lib().us_dgemm(1 if method == "ozaki" else 0, slices, 1 if symmetric else 0, A.shape[0], B.shape[0],
                            A.shape[1], A.ctypes.data, B.ctypes.data, Cm.ctypes.data, C.byref(ms)))
    return (Cm, ms.value) if with_time else Cm


def device_stream(device: int = -1) -> int:
    """The engine's cudaStream_t on `device` (as an int handle)."""
    h = C.c_void_p()
    _check(N.lib().us_device_stream(device, C.byref(h)))
    return h.value or 0


def graph_replays(device: int = -1) -> int:
    """Evaluations on `device` that ran as a replayed CUDA graph so far."""
    c = N.u64()
    _check(N.lib().us_graph_replays(device, C.byref(c)))
    return int(c.value)


def profile(enable: bool = True, reset: bool = True, device: int = -1) -> dict:
    """Reads (and optionally resets) kernel-class event timings, then sets the
    profiling switch. Returns {'gemm_ms','stream_ms','other_ms', '*_groups'}."""
    ms = (N.f64 * 3)()
    groups = (N.u64 * 3)()
    _check(N.lib().us_profile(device, 1 if enable else 0, 1 if reset else 0, ms, groups))
    return {"gemm_ms": ms[0], "stream_ms": ms[1], "other_ms": ms[2],
            "gemm_groups": groups[0], "stream_groups": groups[1], "other_groups": groups[2]}


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(N.lib().us_nccl_unique_id(buf))
    return buf.raw


def nccl_init(device: int, rank: int, world_size: int, uid: bytes) -> None:
    """Creates the engine's NCCL communicator for row sharding on `device`."""
    buf = C.create_string_buffer(bytes(uid), 128)
    _check(N.lib().us_nccl_init(device, rank, world_size, buf))


def device_count() -> int:
    c = N.i32()
    _check(N.lib().us_device_count(C.byref(c)))
    return c.value
