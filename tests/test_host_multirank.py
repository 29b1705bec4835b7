"""Host-side multi-rank logic on CPU (no GPU): rank coordinates, the NCCL communicator
plan of an n x P x D job, and a world-size-2 gloo run of the rank/uid/data-split
plumbing the executor does before it touches NCCL."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_03791_b200 import ModelSpec, ParallelConfig, TaskKind, generate, make_placement
from paper_2402_03791_b200.engine.executor import comm_plan, rank_coords


@pytest.mark.parametrize("n,P,D", [(1, 1, 1), (1, 2, 4), (1, 4, 2), (1, 8, 1), (2, 2, 2), (2, 1, 4), (4, 2, 1)])
def test_rank_coords_bijective(n, P, D):
    seen = {rank_coords(r, n, P, D) for r in range(n * P * D)}
    assert seen == {(a, b, c) for a in range(n) for b in range(P) for c in range(D)}
    with pytest.raises(ValueError):
        rank_coords(n * P * D, n, P, D)


@pytest.mark.parametrize("n,P,D", [(1, 2, 2), (1, 2, 4), (1, 4, 2), (2, 2, 2), (2, 1, 4), (4, 2, 1), (1, 1, 8)])
def test_comm_plan_keys_unique_per_rank(n, P, D):
    """A rank looks communicators up by node-local key: it must belong to at most one
    group per key, groups must stay inside one node (except "inter")."""
    plan = comm_plan(n, P, D)
    for r in range(n * P * D):
        keys = [k for k, ranks in plan if r in ranks]
        assert len(keys) == len(set(keys)), (r, keys)
        node, p, z = rank_coords(r, n, P, D)
        if D > 1:
            assert ("ag", p) in keys and ("rs", p) in keys
        assert (("inter",) in keys) == (n > 1)
    for k, ranks in plan:
        nodes = {rank_coords(x, n, P, D)[0] for x in ranks}
        if k[0] == "inter":
            assert len(nodes) == n and len({rank_coords(x, n, P, D)[1:] for x in ranks}) == 1
        else:
            assert len(nodes) == 1
        assert len(ranks) == len(set(ranks))


@pytest.mark.parametrize("P,V", [(2, 2), (4, 1), (4, 2), (8, 1)])
def test_comm_plan_covers_schedule_p2p(P, V):
    """Every cross-device activation / gradient hand-off the schedule implies
    (F(s)->F(s+1), B(s+1)->B(s); `schedules.py:115-124`) has its directed channel."""
    model = ModelSpec(num_layers=8 * V, hidden_size=256, seq_len=128)
    cfg = ParallelConfig(pp_size=P, dp_size=2, microbatches=2 * P, unit_size=2 * P, stages_per_device=V)
    pl = make_placement(cfg, model)
    sched = generate(model, cfg, pl)
    keys = {k for k, _ in comm_plan(1, P, 2)}
    for a, b in sched.edges:
        if a.device == b.device:
            continue
        if a.kind is TaskKind.F and b.kind is TaskKind.F:
            assert all(("act", a.device, b.device, z) in keys for z in range(2))
        if a.kind is TaskKind.B and b.kind in (TaskKind.B, TaskKind.W):
            assert all(("grad", a.device, b.device, z) in keys for z in range(2))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, P, D, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = comm_plan(n, P, D)
        # rank 0 mints one id per communicator and broadcasts them (executor._init_comms)
        uids = [bytes([i % 256]) * 128 for i in range(len(plan))] if rank == 0 else None
        obj = [uids]
        dist.broadcast_object_list(obj, src=0)
        mine = {k: uid for (k, ranks), uid in zip(plan, obj[0]) if rank in ranks}
        node, p, z = rank_coords(rank, n, P, D)
        dp_index = node * D + z
        # every data-parallel slice of the global batch is consumed by exactly one (node, z)
        # per pipeline rank: gather (p, dp_index) from all ranks
        got = [None] * world
        dist.all_gather_object(got, (p, dp_index, sorted(map(str, mine))))
        out[rank] = got
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,P,D", [(2, 1, 1), (1, 2, 1), (1, 1, 2)])
def test_gloo_world2_plumbing(n, P, D):
    world = n * P * D
    assert world == 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, P, D, out), nprocs=world, join=True)
    got = out[0]
    assert got == out[1]
    for p in range(P):
        assert sorted(dp for pp, dp, _ in got if pp == p) == list(range(n * D))
    # both ranks joined the same set of 2-rank communicators
    assert got[0][2] == got[1][2] and len(got[0][2]) == {(2, 1, 1): 1, (1, 2, 1): 4, (1, 1, 2): 2}[(n, P, D)]
