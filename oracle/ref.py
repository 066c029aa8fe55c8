"""ctypes driver of the reference library compiled from /root/reference
sources (oracle/Makefile -> oracle/_ref/libustats_ref.so).

TEST INFRASTRUCTURE ONLY: the checker for parity tests and the timed CPU
baseline of bench.py (`--impl reference`, `cpu_baseline`). Entry points are
documented in oracle/ref_capi.cpp.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent / "_ref" / "libustats_ref.so"
_lib = None


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise FileNotFoundError(f"{LIB} not built (make -C oracle)")
        _lib = C.CDLL(str(LIB))
        I32P, F64P = C.POINTER(C.c_int), C.POINTER(C.c_double)
        common = [C.c_int, C.c_int, I32P, I32P, C.POINTER(C.c_void_p), C.c_int]
        _lib.ref_u_statistic.argtypes = common + [C.c_int, C.c_uint64, F64P, F64P]
        _lib.ref_v_statistic.argtypes = common + [C.c_int, C.c_uint64, F64P, F64P]
        _lib.ref_u_statistic_unsparsified.argtypes = common + [C.c_int, C.c_uint64, F64P, F64P]
        _lib.ref_restricted_v.argtypes = common + [I32P, C.c_int, F64P]
        _lib.ref_u_brute_force.argtypes = common + [F64P]
        _lib.ref_u_terms.argtypes = common + [C.c_int, C.c_uint64, C.c_int, I32P, I32P,
                                              C.POINTER(C.c_longlong), F64P, F64P]
        _lib.ref_einsum.argtypes = [C.c_int, I32P, I32P, C.POINTER(C.c_void_p), C.c_int, C.c_int, I32P,
                                    C.c_int, F64P, F64P]
        _lib.ref_optimize_order.argtypes = [C.c_int, I32P, I32P, I32P, I32P]
        _lib.ref_u_statistic_data.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64, F64P, F64P]
        _lib.ref_complexity_report.argtypes = [C.c_int, I32P, I32P, C.c_int, I32P, C.POINTER(C.c_uint64),
                                               C.POINTER(C.c_uint64), C.c_char_p, C.c_int]
        _lib.ref_dcov_squared.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, F64P]
        _lib.ref_hoif_tau.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, F64P]
        _lib.ref_motif_count.argtypes = [C.c_int, C.c_int, I32P, C.c_char_p, C.c_int, C.POINTER(C.c_longlong)]
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


def _enc(signature):
    lens = [len(t) for t in signature]
    idx = [s for t in signature for s in t]
    return (len(lens), (C.c_int * len(lens))(*lens), (C.c_int * max(1, len(idx)))(*idx))


class _Fx:
    def __init__(self, factors):
        self.keep, ptrs, seen = [], [], {}
        for f in factors:
            if id(f) in seen:
                ptrs.append(ptrs[seen[id(f)]])
                continue
            a = np.ascontiguousarray(f, dtype=np.float64)
            self.keep.append(a)
            seen[id(f)] = len(ptrs)
            ptrs.append(a.ctypes.data)
        self.ptrs = (C.c_void_p * len(ptrs))(*ptrs)
        self.n = int(np.shape(factors[0])[0])


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"reference failed ({rc}): {lib().ref_last_error().decode()}")


STAT_KEYS = ["tensorize_seconds", "contract_seconds", "einsum_calls", "partitions_enumerated",
             "partitions_evaluated", "multiply_adds", "peak_intermediate_entries"]


def u_statistic(factors, signature, m, threads=0, cap=0):
    K, L, I = _enc(signature)
    fx = _Fx(factors)
    out = C.c_double()
    st = (C.c_double * 7)()
    _check(lib().ref_u_statistic(m, K, L, I, fx.ptrs, fx.n, threads, cap, C.byref(out), st))
    return out.value, dict(zip(STAT_KEYS, list(st)))


def v_statistic(factors, signature, m, threads=0):
    K, L, I = _enc(signature)
    fx = _Fx(factors)
    out = C.c_double()
    st = (C.c_double * 7)()
    _check(lib().ref_v_statistic(m, K, L, I, fx.ptrs, fx.n, threads, 0, C.byref(out), st))
    return out.value


def u_statistic_unsparsified(factors, signature, m, threads=0):
    K, L, I = _enc(signature)
    fx = _Fx(factors)
    out = C.c_double()
    st = (C.c_double * 7)()
    _check(lib().ref_u_statistic_unsparsified(m, K, L, I, fx.ptrs, fx.n, threads, 0, C.byref(out), st))
    return out.value


def restricted_v(factors, signature, m, rgs, threads=1):
    K, L, I = _enc(signature)
    fx = _Fx(factors)
    out = C.c_double()
    _check(lib().ref_restricted_v(m, K, L, I, fx.ptrs, fx.n, (C.c_int * m)(*rgs), threads, C.byref(out)))
    return out.value


def u_brute_force(factors, signature, m):
    K, L, I = _enc(signature)
    fx = _Fx(factors)
    out = C.c_double()
    _check(lib().ref_u_brute_force(m, K, L, I, fx.ptrs, fx.n, C.byref(out)))
    return out.value


def u_terms(factors, signature, m, threads=1, cap=0, max_terms=4140):
    K, L, I = _enc(signature)
    fx = _Fx(factors)
    cnt = C.c_int()
    rgs = (C.c_int * (max_terms * m))()
    mu = (C.c_longlong * max_terms)()
    v = (C.c_double * max_terms)()
    madds = (C.c_double * max_terms)()
    _check(lib().ref_u_terms(m, K, L, I, fx.ptrs, fx.n, threads, cap, max_terms, C.byref(cnt), rgs, mu, v, madds))
    T = cnt.value
    return (np.array(rgs[:T * m], dtype=np.int32).reshape(T, m), np.array(mu[:T], dtype=np.int64),
            np.array(v[:T]), np.array(madds[:T]))


def einsum(tensors, inputs, output=(), threads=1):
    K, L, I = _enc(inputs)
    arrays = [np.ascontiguousarray(t, dtype=np.float64) for t in tensors]
    ptrs = (C.c_void_p * K)(*[a.ctypes.data for a in arrays])
    n = next((a.shape[0] for a in arrays if a.ndim), 1)
    out = np.zeros((n,) * len(output))
    madds = C.c_double()
    O = (C.c_int * max(1, len(output)))(*output)
    _check(lib().ref_einsum(K, L, I, ptrs, n, len(output), O, threads,
                            out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(madds)))
    return out, madds.value


def optimize_order(inputs):
    K, L, I = _enc(inputs)
    ids = len({s for t in inputs for s in t})
    out = (C.c_int * ids)()
    w = C.c_int()
    _check(lib().ref_optimize_order(K, L, I, out, C.byref(w)))
    return list(out), w.value


def u_statistic_data(spec, data, threads=0, cap=0):
    """The reference's u_statistic on a data kernel: components evaluated per
    entry by its own tensorize (rbf / proj / hoif / prod2 specs)."""
    x = np.ascontiguousarray(data, dtype=np.float64)
    if x.ndim == 1:
        x = x.reshape(-1, 1)
    out = C.c_double()
    st = (C.c_double * 7)()
    _check(lib().ref_u_statistic_data(spec.encode(), C.c_void_p(x.ctypes.data), x.shape[0], x.shape[1], threads, cap,
                                      C.byref(out), st))
    return out.value, dict(zip(STAT_KEYS, list(st)))


def complexity_report(signature, extent):
    """The reference's complexity_report as a dict (same keys as the engine's)."""
    K, L, I = _enc(signature)
    ints = (C.c_int * 8)()
    counts = (C.c_uint64 * 2)()
    hist = (C.c_uint64 * 16)()
    buf = C.create_string_buffer(512)
    _check(lib().ref_complexity_report(K, L, I, int(extent), ints, counts, hist, buf, 512))
    return {"index_count": ints[0], "extent": ints[1], "graph_vertices": ints[2], "graph_edges": ints[3],
            "treewidth_lower": ints[4], "treewidth_upper": ints[5],
            "treewidth_exact": None if ints[6] < 0 else ints[6], "max_quotient_width": ints[7],
            "bell_count": counts[0], "sparsified_count": counts[1],
            "count_by_width": {w: int(c) for w, c in enumerate(hist) if c}, "flops_estimate": buf.value.decode()}


def dcov_squared(x, y, threads=0):
    """The reference's dcov_squared on paired samples (rows = observations)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    x = x.reshape(x.shape[0], -1)
    y = y.reshape(y.shape[0], -1)
    out = C.c_double()
    _check(lib().ref_dcov_squared(x.ctypes.data, x.shape[1], y.ctypes.data, y.shape[1], x.shape[0], threads,
                                  C.byref(out)))
    return out.value


def hoif_tau(m, k, data, threads=0):
    """The reference's hoif_tau with truncation_phi(k) on rows [A, Y, Z...]."""
    x = np.ascontiguousarray(data, dtype=np.float64)
    out = C.c_double()
    _check(lib().ref_hoif_tau(m, k, x.ctypes.data, x.shape[0], x.shape[1], threads, C.byref(out)))
    return out.value


def motif_count(n, edges, motif_id, threads=0):
    """The reference's motif_count on the graph over vertices 0..n-1."""
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    out = C.c_longlong()
    _check(lib().ref_motif_count(int(n), e.shape[0], e.ctypes.data_as(C.POINTER(C.c_int)), motif_id.encode(),
                                 threads, C.byref(out)))
    return out.value
