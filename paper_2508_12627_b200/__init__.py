"""B200-native exact U-statistics by partition-lattice tensor contraction.

Host planning (partition lattice, Möbius weights, treewidth-optimal orders)
in C++; V-term contractions as sm_100a kernels (FP64 DMMA GEMMs, fused
broadcast-product-reduce streams) behind the C-ABI in include/ustats_b200.h.
"""
from .api import (  # noqa: F401
    Config, UStatsError, UTerms, bell_number, combine_terms, device_count, device_stream, einsum,
    profile, nccl_init, nccl_unique_id, graph_replays,
    eliminate_index, kernel_tensors, optimize_order, plan_summary, plan_terms, restricted_v_tensors, survivors, treewidth,
    ComplexityReport, chain_signature, complexity_report, dgemm,
    u_statistic, u_statistic_batch, u_statistic_tensors, u_statistic_unsparsified_tensors, u_terms,
    v_statistic, hoif_tau, dcov_squared, motif_count, MOTIF_IDS,
    v_statistic_tensors,
)
from ._native import LIB_PATH, lib  # noqa: F401
