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


# ---- row sharding (shard.cpp): the plan every rank derives on its own

def _shard_plan(name, n, world, rank):
    import paper_2508_12627_b200 as us
    from paper_2508_12627_b200.workloads import CONFIGS
    w = CONFIGS[name]
    sig = [list(t) for t in w.signature]
    cfg = us.Config(memory_cap_entries=2 ** 40, shard_rows=True, world_size=world, rank=rank)
    txt, _ = us.plan_summary(sig, w.m, n, cfg)
    return txt[txt.index("-- shard plan"):].splitlines()[1:]


def _parse(lines):
    head = dict(kv.split("=") for kv in lines[0].split())
    steps = []
    for ln in lines[1:]:
        parts = ln.split()
        colls = [p for p in parts if p.startswith(("pre:", "post:"))]
        rows = next((p for p in parts if p.startswith("rows=")), None)
        pieces = next((p for p in parts if p.startswith("pieces=")), None)
        steps.append({"op": parts[1], "mode": parts[3], "colls": colls, "rows": rows, "pieces": pieces})
    return head, steps


def _plan_worker(rank, world, port, name, n, out):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plans = [None] * world
    dist.all_gather_object(plans, _shard_plan(name, n, world, rank))
    out[rank] = plans
    dist.destroy_process_group()


@pytest.mark.parametrize("name,n", [("C5", 65536), ("C4", 1024)])
def test_two_rank_gloo_row_sharding_plans_agree(name, n):
    # each rank plans on its own; over gloo they must agree on every
    # collective (same buffers, same order) and their row slices must
    # partition [0, n) for every row-sharded op
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_plan_worker, args=(world, _free_port(), name, n, out), nprocs=world, join=True)
    plans = [_parse(p) for p in out[0]]
    assert out[0] == out[1]  # both ranks saw the same set of plans
    (h0, s0), (h1, s1) = plans
    assert len(s0) == len(s1) > 0
    for a, b in zip(s0, s1):
        assert (a["op"], a["mode"], a["colls"]) == (b["op"], b["mode"], b["colls"])
        if a["rows"]:
            lo0, hi0 = map(int, a["rows"][6:-1].split(","))
            lo1, hi1 = map(int, b["rows"][6:-1].split(","))
            assert (lo0, hi0, lo1, hi1) == (0, lo1, hi0, n)
    # all-reduces touch vectors and scalars only (no n^2 buffer is ever
    # all-reduced); gathers move row slabs of what a later op reads whole
    colls = [c for s in s0 for c in s["colls"]]
    assert all(int(c.split(":o")[1]) <= 1 for c in colls if ":reduce:" in c)
    assert any(":exchange:" in c for c in colls)


@pytest.mark.parametrize("world", [2, 3, 4, 5, 8])
def test_symmetric_pieces_cover_the_matrix_once(world):
    # the triangle pieces of all ranks, each stored directly and transposed,
    # cover every entry of a symmetric product exactly once, and the block
    # units per rank are balanced
    import re
    n = 1000
    lines = [_shard_plan("C5", n, world, r) for r in range(world)]
    cover = np.zeros((n, n), dtype=np.int32)
    units = []
    for r in range(world):
        step = next(ln for ln in lines[r][1:] if "pieces=" in ln)
        pieces = re.findall(r"\[(\d+),(\d+)\)x\[(\d+),(\d+)\)->(\d+)", step)
        area = 0
        for r0, r1, c0, c1, owner in pieces:
            r0, r1, c0, c1 = map(int, (r0, r1, c0, c1))
            cover[r0:r1, c0:c1] += 1
            if (r0, r1) != (c0, c1):
                cover[c0:c1, r0:r1] += 1
                area += (r1 - r0) * (c1 - c0)
            else:
                area += (r1 - r0) * (c1 - c0) / 2
        units.append(area)
    assert np.all(cover == 1)
    assert max(units) <= 1.02 * min(units) + n
