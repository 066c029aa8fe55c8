"""ctypes binding of ``libustats_b200.so`` (the C-ABI in include/ustats_b200.h).

The shared library is built in-tree by ``build.py``. There is no CPU fallback:
if the library is missing, importing the engine raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libustats_b200.so"

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
P = C.POINTER


class UsConfig(C.Structure):
    _fields_ = [
        ("memory_cap_entries", u64),
        ("threads", i32),
        ("strategy", i32),
        ("exhaustive_index_bound", i32),
        ("exact_treewidth_bound", i32),
        ("device", i32),
        ("rank", i32),
        ("world_size", i32),
        ("flags", i32),
        ("emulate_world", i32),
        ("memory_budget_bytes", u64),
        ("oz_slices", i32),
        ("oz_min_dim", i32),
        ("oz_max_k", i64),
    ]


class UsStats(C.Structure):
    _fields_ = [
        ("tensorize_seconds", f64),
        ("contract_seconds", f64),
        ("einsum_calls", u64),
        ("partitions_enumerated", u64),
        ("partitions_evaluated", u64),
        ("multiply_adds", u64),
        ("peak_intermediate_entries", u64),
        ("executed_gemm_macs", u64),
        ("executed_stream_entries", u64),
        ("gemm_launches", u64),
        ("stream_launches", u64),
        ("shared_hits", u64),
        ("kernel_launches", u64),
        ("emulated_gemm_macs", u64),
        ("int8_tensor_ops", u64),
        ("oz_slices", u64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class UsComplexity(C.Structure):
    _fields_ = [
        ("index_count", i32),
        ("extent", i32),
        ("graph_vertices", i32),
        ("graph_edges", i32),
        ("treewidth_lower", i32),
        ("treewidth_upper", i32),
        ("treewidth_exact", i32),
        ("max_quotient_width", i32),
        ("bell_count", u64),
        ("sparsified_count", u64),
        ("count_by_width", u64 * 16),
    ]


# name -> (restype, argtypes); exactly the declarations of include/ustats_b200.h
SIGNATURES = {
    "us_version": (C.c_char_p, []),
    "us_last_error": (C.c_char_p, []),
    "us_config_default": (None, [P(UsConfig)]),
    "us_u_statistic": (C.c_int, [i32, i32, P(i32), P(i32), P(C.c_void_p), i64, i32, P(UsConfig), P(f64), P(UsStats)]),
    "us_u_terms": (C.c_int, [i32, i32, P(i32), P(i32), P(C.c_void_p), i64, i32, P(UsConfig), i32, P(i32),
                             P(i32), P(i64), P(f64), P(i32), P(f64), P(UsStats)]),
    "us_u_statistic_data": (C.c_int, [C.c_char_p, C.c_void_p, i64, i32, i32, P(UsConfig), P(f64), P(UsStats)]),
    "us_u_statistic_batch": (C.c_int, [i32, P(i32), P(i32), P(i32), P(i32), P(C.c_void_p), i64, i32, P(UsConfig),
                                       P(f64), P(UsStats)]),
    "us_u_statistic_unsparsified": (C.c_int, [i32, i32, P(i32), P(i32), P(C.c_void_p), i64, i32, P(UsConfig),
                                              P(f64), P(UsStats)]),
    "us_v_statistic": (C.c_int, [i32, i32, P(i32), P(i32), P(C.c_void_p), i64, P(UsConfig), P(f64), P(UsStats)]),
    "us_restricted_v": (C.c_int, [i32, i32, P(i32), P(i32), P(C.c_void_p), i64, P(i32), P(UsConfig), P(f64),
                                  P(UsStats)]),
    "us_einsum": (C.c_int, [i32, P(i32), P(i32), P(C.c_void_p), i64, i32, P(i32), P(i32), i32, P(UsConfig),
                            P(f64), P(u64), P(u64), P(i32)]),
    "us_eliminate_index": (C.c_int, [i32, P(i32), P(i32), P(C.c_void_p), i64, i32, P(UsConfig), P(f64), u64,
                                     P(i32), P(i32)]),
    "us_combine_terms": (f64, [i32, P(i64), P(f64)]),
    "us_bell_number": (u64, [i32]),
    "us_survivors": (C.c_int, [i32, i32, P(i32), P(i32), i32, P(i32), P(i32), P(i64), P(u64)]),
    "us_optimize_order": (C.c_int, [i32, P(i32), P(i32), i32, P(i32), P(i32), P(i32)]),
    "us_treewidth": (C.c_int, [i32, i32, P(i32), P(i32), P(i32)]),
    "us_dcov_squared": (C.c_int, [C.c_void_p, i32, C.c_void_p, i32, i64, i32, P(UsConfig), P(f64), P(UsStats)]),
    "us_hoif_tau": (C.c_int, [i32, i32, C.c_void_p, i64, i32, i32, P(UsConfig), P(f64), P(UsStats)]),
    "us_motif_count": (C.c_int, [i64, i64, P(i32), C.c_char_p, P(UsConfig), P(i64), P(UsStats)]),
    "us_dgemm": (C.c_int, [i32, i32, i32, i64, i64, i64, C.c_void_p, C.c_void_p, C.c_void_p, P(f64)]),
    "us_complexity_report": (C.c_int, [i32, P(i32), P(i32), i32, P(UsConfig), P(UsComplexity), C.c_char_p, i32]),
    "us_plan_terms": (C.c_int, [i32, i32, P(i32), P(i32), i64, i32, i32, P(i32), P(i32), P(f64)]),
    "us_plan_summary": (C.c_int, [i32, i32, P(i32), P(i32), i64, P(UsConfig), i32, C.c_char_p, u64, P(u64)]),
    "us_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "us_nccl_init": (C.c_int, [i32, i32, i32, C.c_void_p]),
    "us_device_count": (C.c_int, [P(i32)]),
    "us_device_synchronize": (C.c_int, [i32]),
    "us_device_stream": (C.c_int, [i32, P(C.c_void_p)]),
    "us_graph_replays": (C.c_int, [i32, P(u64)]),
    "us_profile": (C.c_int, [i32, i32, i32, P(f64), P(u64)]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -m paper_2508_12627_b200.build` "
                "(the B200 engine has no CPU fallback)")
        handle = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib
