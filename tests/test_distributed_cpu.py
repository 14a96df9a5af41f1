"""Host-side logic of the multi-GPU path with world_size 2 on CPU (gloo):
shard planning, NCCL unique-id exchange over torch.distributed, assembly of
the sharded T, and the winner rule of the per-step record exchange (value
desc, GLOBAL index asc — the reference's strict '>' scan,
workspace.cpp:107-113, must survive sharding), run by the library's own code
(rbd_shard_pick: csrc/rbd_select.h, the function the device kernels call)."""
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
    """(value, global index) of the winner, by the library's rule."""
    v, j, owner = rd.pick_winner(records)
    return None if owner < 0 else (v, j)


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
        # the greedy loop's steps over two shards: every rank scans its own
        # columns of the oracle's residual bookkeeping (workspace.cpp:52-53,
        # 107-113) and the exchanged records pick the whole-matrix argmax
        import oracle
        X = oracle.random_matrix(40, 23, 77)
        X[:, 17] = X[:, 4]                       # an exact tie across the two shards
        ref = oracle.decompose(X, 6)
        plan2 = rd.plan_shards(23, world)
        o2, n2 = plan2.offsets[rank], plan2.n_locals[rank]
        r_all = oracle.column_sq(X)
        steps_ok = True
        for kk in range(ref.d - 1):
            r_all = np.maximum(r_all - ref.T[kk] * ref.T[kk], 0.0)
            loc = r_all[o2:o2 + n2]
            lj = int(np.argmax(loc))
            mine = torch.tensor([loc[lj], float(o2 + lj)], dtype=torch.float64)
            got = [torch.empty(2, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(got, mine)
            v, j, owner = rd.pick_winner([(float(t[0]), int(t[1])) for t in got])
            steps_ok = steps_ok and j == ref.selected[kk + 1] and owner == plan2.owner(j)
        q.put((rank, plan, len(uid), ids[0] == ids[-1], bool(torch.equal(Tg, T)), win, steps_ok))
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
    for rank, plan, uid_len, same_uid, t_ok, win, steps_ok in out:
        assert plan.offsets == (0, 6) and plan.n_locals == (6, 5)
        assert uid_len == 128 and same_uid
        assert t_ok
        assert win == (7.0, 3)
        assert steps_ok


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
    assert rd.pick_winner([(-2.0, -1), (-2.0, -1)])[2] == -1
    assert rd.pick_winner([(3.0, 9), (3.0, 9 + 2**40)]) == (3.0, 9, 0)
