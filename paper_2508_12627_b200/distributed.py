"""Multi-GPU evaluation: one process per GPU.

Two schemes (BASELINE north_star: "the outermost summed index is row-sharded
and independent V-terms are distributed"):

* ``mode="terms"`` — each rank contracts only the survivors the host plan
  assigns it (LPT on n^(width+1), plan_terms / us_plan_terms); per-term
  values meet in ONE all-reduce (NCCL over NVLink on GPUs, gloo in the CPU
  tests), then every rank applies the reference's combination
  (engine.cpp:47-104). Ownership is one-hot, so the all-reduce is exact.
* ``mode="rows"`` — every rank records the same optimized program and runs a
  slice of every op (a contiguous range of each GEMM's tile list, a range of
  each reduction's leading index) into zeroed outputs; the engine's own NCCL
  communicator all-reduces each materialized output and, at the end, the
  vector of partial V-terms. Scales the shared GEMMs of the cross-term plan
  (C5: 8 GEMMs of 65536^3), which term sharding cannot split.
"""
from __future__ import annotations

from dataclasses import replace
from typing import Callable

import numpy as np

from .api import Config, UTerms, combine_terms, nccl_init, nccl_unique_id, u_terms


def sharded_u_statistic(factors, signature, m: int, config: Config | None = None, group=None,
                        evaluate: Callable | None = None, device=None):
    """Returns (U, per-rank UTerms). ``evaluate(factors, signature, m, cfg)``
    defaults to the GPU engine's u_terms; tests substitute a CPU evaluator."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    cfg = replace(config or Config(), rank=rank, world_size=world)
    terms: UTerms = (evaluate or u_terms)(factors, signature, m, cfg)
    backend = dist.get_backend(group)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    v = torch.from_numpy(np.ascontiguousarray(terms.v)).to(device)
    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    v_all = v.cpu().numpy()
    return combine_terms(terms.mu, v_all), terms


def init_row_sharding(device: int, group=None) -> None:
    """Creates the engine's NCCL communicator on every rank (id from rank 0,
    broadcast over torch.distributed)."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    box = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    nccl_init(device, rank, world, box[0])


def row_sharded_u_statistic(factors, signature, m: int, config: Config | None = None, group=None):
    """U with every op row-sharded (init_row_sharding first). Every rank
    returns the same value: the engine all-reduces the partial V-terms."""
    import torch.distributed as dist

    cfg = replace(config or Config(), rank=dist.get_rank(group), world_size=dist.get_world_size(group),
                  shard_rows=True)
    terms = u_terms(factors, signature, m, cfg)
    return terms.value, terms
