"""Sharded (multi-GPU) path on one B200: the same kernels and exchange protocol
(16-byte record allgather, -0.0-padded payload allreduce, CUDA-graph replay of
8 steps) with R column shards stepped in lockstep in one process. Results must
be bit-identical to the single-GPU loop for any R (per-column
sums depend on m only; the exchanges move bits, never round them)."""
import numpy as np
import pytest

import oracle
import paper_1503_05947_b200 as rbd
from paper_1503_05947_b200 import configs, distributed

pytestmark = pytest.mark.gpu


def dev(a, cuda):
    import torch
    return torch.as_tensor(np.asfortranarray(a).T.copy(), device=cuda).t()


def single(X, d_max, eps=0.0, **kw):
    g = rbd.decompose(X, d_max=d_max, eps_r=eps, **kw)
    return g.Y.cpu().numpy(), g.T.cpu().numpy(), g.d, g.selected, g.residual_history


def check_same(ref, Ys, T, d, sel, hist):
    Yr, Tr, dr, selr, histr = ref
    assert d == dr and sel == selr and hist == histr
    for Y in Ys:
        assert np.array_equal(Y.cpu().numpy(), Yr)
    assert np.array_equal(T.cpu().numpy(), Tr)


@pytest.mark.parametrize("R", [1, 2, 3, 4, 8])
def test_c0_bitwise_across_shards(cuda, R):
    X = dev(configs.c0_matrix(), cuda)
    ref = single(X, 64, 1e-6)
    check_same(ref, *distributed.decompose_virtual(X, R, 64, 1e-6)[:5])


@pytest.mark.parametrize("R", [2, 5])
def test_multichunk_rows_bitwise(cuda, R):
    X = dev(oracle.random_matrix(9000, 210, 4), cuda)
    ref = single(X, 40)
    check_same(ref, *distributed.decompose_virtual(X, R, 40)[:5])


def test_uneven_shards_and_start_in_last(cuda):
    X = dev(oracle.random_matrix(700, 200, 5), cuda)
    ref = single(X, 30, start_column=199)
    out = distributed.decompose_virtual(X, 3, 30, n_locals=[1, 100, 99], start_column=199)
    check_same(ref, *out[:5])
    assert out[3][0] == 199


def test_breakdown_and_oracle_parity(cuda):
    x = oracle.random_low_rank(40, 30, 5, 210)
    X = dev(x, cuda)
    Ys, T, d, sel, hist, _ = distributed.decompose_virtual(X, 4, 30)
    assert d == 5
    r = oracle.decompose(x, 30)
    assert sel == r.selected
    assert np.abs(Ys[0].cpu().numpy() - r.Y).max() < 1e-10


def test_ties_across_shards_smallest_global_index(cuda):
    # identical columns in different shards: the smallest global index must win
    x = oracle.random_matrix(64, 12, 6)
    x[:, 9] = x[:, 2] * 3.0
    x[:, 5] = x[:, 2] * 3.0
    X = dev(x, cuda)
    ref = single(X, 6)
    check_same(ref, *distributed.decompose_virtual(X, 3, 6)[:5])


def test_sharded_gating(cuda):
    with pytest.raises(rbd.DegenerateInput):
        distributed.decompose_virtual(dev(np.zeros((8, 6)), cuda), 2, 3)
    x = oracle.random_matrix(8, 6, 1)
    x[2, 4] = np.nan
    with pytest.raises(rbd.InvalidArgument):
        distributed.decompose_virtual(dev(x, cuda), 2, 3)
    with pytest.raises(rbd.InvalidArgument):
        distributed.decompose_virtual(dev(oracle.random_matrix(8, 6, 1), cuda), 2, 7)


def test_nccl_world1_matches_single_gpu(cuda):
    """The real NCCL exchange (communicator of size 1) gives the single-GPU bits."""
    import ctypes as C
    from paper_1503_05947_b200._lib import check, load_library
    X = dev(oracle.random_matrix(5000, 300, 8), cuda)
    ref = single(X, 50)
    ctx = rbd.Context(0)
    buf = C.create_string_buffer(128)
    check(load_library().rbd_comm_unique_id(buf))
    distributed.init_comm(ctx, 0, 1, bytes(buf.raw))
    plan = distributed.plan_shards(300, 1)
    r = distributed.decompose_sharded(X, plan, 0, 50, ctx=ctx)
    assert r.result.reserved == 1                    # NCCL calls captured in the step graph
    assert r.d == ref[2] and r.selected == ref[3] and r.residual_history == ref[4]
    assert np.array_equal(r.Y.cpu().numpy(), ref[0])
    assert np.array_equal(r.T_local.cpu().numpy(), ref[1])
    ctx.close()


@pytest.mark.parametrize("R", [1, 3])
def test_graph_replay_and_eager_steps_agree(cuda, monkeypatch, R):
    """The steps are replayed from a CUDA graph (result.reserved == 1); the eager
    host-driven loop (RBD_SHARD_GRAPH=0) gives the same bits, including a stop
    in the middle of a replay (d = 13 is not a multiple of 8)."""
    X = dev(oracle.random_matrix(3000, 120, 12), cuda)
    ref = single(X, 13)
    g = distributed.decompose_virtual(X, R, 13)
    assert g[5].reserved == 1
    check_same(ref, *g[:5])
    monkeypatch.setenv("RBD_SHARD_GRAPH", "0")
    e = distributed.decompose_virtual(X, R, 13)
    assert e[5].reserved == 0
    check_same(ref, *e[:5])


def test_signed_zero_columns_survive_the_payload_allreduce(cuda):
    """The owner's payload travels through a sum with -0.0 from every other rank:
    exact for every value, -0.0 entries of x included."""
    x = oracle.random_matrix(256, 24, 13)
    x[::3, :] = -0.0
    X = dev(x, cuda)
    ref = single(X, 10)
    bits = lambda a: np.asarray(a).view(np.int64)   # noqa: E731  (tells -0.0 from +0.0)
    for R in (2, 4):
        out = distributed.decompose_virtual(X, R, 10)
        check_same(ref, *out[:5])
        for Y in out[0]:
            assert np.array_equal(bits(Y.cpu().numpy()), bits(ref[0]))
        assert np.array_equal(bits(out[1].cpu().numpy()), bits(ref[1]))
