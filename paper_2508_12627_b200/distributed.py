"""Multi-GPU evaluation: one process per GPU, V-terms sharded over ranks.

Each rank contracts only the survivors the host plan assigns it (LPT on
n^(width+1), plan_terms / us_plan_terms); per-term values meet in ONE
all-reduce (NCCL over NVLink on GPUs, gloo in the CPU tests), after which
every rank applies the reference's combination (engine.cpp:47-104) to the
same vector. Every term has exactly one owner, so the all-reduce adds zeros
to one non-zero and is exact: the result is bit-identical to 1 GPU given
identical per-term values.
"""
from __future__ import annotations

from dataclasses import replace
from typing import Callable

import numpy as np

from .api import Config, UTerms, combine_terms, u_terms


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
