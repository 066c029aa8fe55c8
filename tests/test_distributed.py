"""World-size-2 gloo test of the multi-rank path: term ownership from the
engine's host plan, per-rank evaluation of owned terms, one all-reduce, the
reference combination. On CPU the per-term evaluator is the oracle (the GPU
runs the same plumbing with the CUDA engine)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, n, out):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ustats_np as O
    import paper_2508_12627_b200 as us
    from paper_2508_12627_b200.api import UTerms
    from paper_2508_12627_b200.distributed import sharded_u_statistic
    from paper_2508_12627_b200.workloads import generate

    factors, sig, m, _ = generate(name, n)

    def cpu_evaluate(factors, sig, m, cfg):
        owner, _ = us.plan_terms(sig, m, n, cfg.world_size)
        _, rows = O.u_statistic(factors, sig, m)
        v = np.array([r[2] if owner[t] == cfg.rank else 0.0 for t, r in enumerate(rows)])
        return UTerms(0.0, np.array([r[0] for r in rows]), np.array([r[1] for r in rows]), v, owner)

    u, terms = sharded_u_statistic(factors, sig, m, us.Config(), evaluate=cpu_evaluate)
    out[rank] = (u, int((terms.owner == rank).sum()))
    dist.destroy_process_group()


@pytest.mark.parametrize("name,n", [("C2", 48), ("C5", 96)])
def test_two_rank_gloo_matches_single_rank(name, n):
    from oracle import ustats_np as O
    from paper_2508_12627_b200.workloads import generate
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), name, n, out), nprocs=world, join=True)
    factors, sig, m, _ = generate(name, n)
    u_single, rows = O.u_statistic(factors, sig, m)
    assert out[0][0] == out[1][0]  # every rank combines the same vector
    assert out[0][0] == u_single  # one-hot ownership: the all-reduce is exact
    assert out[0][1] + out[1][1] == len(rows)
    assert out[0][1] > 0 and out[1][1] > 0
