"""Host-side logic of the multi-GPU path with world_size 2 on CPU (gloo):
shard planning, NCCL unique-id exchange over torch.distributed, assembly of
the sharded T, and the winner-selection rule of the payload protocol
(value desc, GLOBAL index asc — the reference's strict '>' scan,
workspace.cpp:107-113, must survive sharding)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1503_05947_b200 import distributed as rd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def select_winner(records):
    """The k_shard_select rule on gathered (value, global index) records."""
    best = None
    for v, j in records:
        if j < 0:
            continue
        if best is None or v > best[0] or (v == best[0] and j < best[1]):
            best = (v, j)
    return best


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 11
        plan = rd.plan_shards(n, world)
        uid = rd.exchange_unique_id(rank)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        # the sharded T assembles to the global T
        T = torch.arange(3 * n, dtype=torch.float64).reshape(3, n)
        o, nl = plan.offsets[rank], plan.n_locals[rank]
        Tg = rd.assemble_T(T[:, o:o + nl].clone(), plan)
        # protocol: each rank's local best record with global indices; an exact
        # tie across ranks (global columns 3 and 8) must go to index 3
        r = np.array([0.5, 0.1, 0.2, 7.0, 0.3, 1.0, 2.0, 0.0, 7.0, 6.9, 0.4])
        loc = r[o:o + nl]
        lj = int(np.argmax(loc))   # first max within the shard
        rec = torch.tensor([loc[lj], float(o + lj)], dtype=torch.float64)
        recs = [torch.empty(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(recs, rec)
        win = select_winner([(float(t[0]), int(t[1])) for t in recs])
        q.put((rank, plan, len(uid), ids[0] == ids[-1], bool(torch.equal(Tg, T)), win))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_protocol():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, plan, uid_len, same_uid, t_ok, win in out:
        assert plan.offsets == (0, 6) and plan.n_locals == (6, 5)
        assert uid_len == 128 and same_uid
        assert t_ok
        assert win == (7.0, 3)


def test_plan_shards():
    p = rd.plan_shards(65536, 8, block=8192)
    assert p.offsets == tuple(8192 * r for r in range(8)) and set(p.n_locals) == {8192}
    p = rd.plan_shards(10, 3)
    assert p.n_locals == (4, 3, 3) and p.offsets == (0, 4, 7)
    assert p.owner(4) == 1 and p.local(9) == (2, 2)
    with pytest.raises(ValueError):
        rd.plan_shards(10, 3, block=3)


def test_select_rule():
    assert select_winner([(1.0, 5), (1.0, 2), (0.5, 1)]) == (1.0, 2)
    assert select_winner([(-2.0, -1), (0.0, 7)]) == (0.0, 7)
