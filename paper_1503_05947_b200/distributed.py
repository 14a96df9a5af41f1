"""Multi-GPU RBD: one process per GPU, X sharded by
contiguous column blocks, Y replicated.

Host-side plumbing lives here (shard plan, NCCL unique-id exchange over
torch.distributed, result assembly); the per-step exchange (one payload
allgather) runs inside the C library over NCCL (rbd_decompose_sharded).
``decompose_virtual`` runs the same kernels and protocol with R shards in one
process on one device (payload exchange by device copies) — the way the
sharded path is tested for bitwise identity on a single GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from ._lib import Context, Result, check, default_context, load_library
from .api import _col_major_torch, make_config


@dataclass(frozen=True)
class ShardPlan:
    """Contiguous column blocks: rank r owns global columns [offset, offset+n_local)."""
    n_global: int
    offsets: tuple
    n_locals: tuple

    @property
    def world(self) -> int:
        return len(self.offsets)

    def owner(self, j: int) -> int:
        for r, (o, nl) in enumerate(zip(self.offsets, self.n_locals)):
            if o <= j < o + nl:
                return r
        raise IndexError(j)

    def local(self, j: int):
        r = self.owner(j)
        return r, j - self.offsets[r]


def plan_shards(n: int, world: int, block: Optional[int] = None) -> ShardPlan:
    """Balanced contiguous column blocks (the first n % world ranks get one
    more column), or fixed blocks of ``block`` columns (C3: 8192 per GPU)."""
    if world < 1 or n < 1:
        raise ValueError("plan_shards: need n >= 1 and world >= 1")
    if block is not None:
        sizes = [max(0, min(block, n - r * block)) for r in range(world)]
        if sum(sizes) != n:
            raise ValueError("plan_shards: block * world must cover n")
    else:
        base, extra = divmod(n, world)
        sizes = [base + (1 if r < extra else 0) for r in range(world)]
    offs, o = [], 0
    for s in sizes:
        offs.append(o)
        o += s
    return ShardPlan(n, tuple(offs), tuple(sizes))


def exchange_unique_id(rank: int, group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; everyone receives it through
    torch.distributed (any backend, gloo included)."""
    import torch.distributed as dist
    obj: List[Optional[bytes]] = [None]
    if rank == 0:
        buf = C.create_string_buffer(128)
        check(load_library().rbd_comm_unique_id(buf))
        obj[0] = bytes(buf.raw)
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def pick_winner(records):
    """The per-step winner rule of the record exchange, run by the library's own
    code (rbd_shard_pick, csrc/rbd_select.h — the same function the device
    kernels call): records = [(best residual, global index or -1)] per rank.
    Returns (value, global index, owner rank); owner -1 when nobody has one."""
    recs = np.zeros(2 * len(records))
    for r, (v, j) in enumerate(records):
        recs[2 * r] = float(v)
        recs[2 * r + 1] = np.array([int(j)], dtype=np.int64).view(np.float64)[0]
    bv, bj, own = C.c_double(), C.c_int64(), C.c_int()
    check(load_library().rbd_shard_pick(recs.ctypes.data_as(C.c_void_p), len(records),
                                        C.byref(bv), C.byref(bj), C.byref(own)))
    return bv.value, bj.value, own.value


def init_comm(ctx: Context, rank: int, world: int, uid: bytes) -> None:
    check(load_library().rbd_ctx_init_comm(ctx.handle, rank, world, uid))


@dataclass
class ShardedModel:
    Y: object                    # m x d (replicated on every rank)
    T_local: object              # d x n_local (this rank's columns)
    d: int
    selected: List[int]          # global column indices
    residual_history: List[float]
    result: Result
    plan: ShardPlan
    rank: int


def decompose_sharded(X_local, plan: ShardPlan, rank: int, d_max: int, eps_r: float = 0.0,
                      ctx: Optional[Context] = None, **cfg_kw) -> ShardedModel:
    """rbd::decompose over the column shards of all ranks (NCCL). Call
    ``init_comm`` on ``ctx`` first. X_local: m x n_local column-major CUDA tensor."""
    import torch
    lib = load_library()
    ctx = ctx or default_context(X_local.device.index or 0)
    cfg = make_config(d_max, eps_r, **cfg_kw)
    xc, ldx = _col_major_torch(X_local)
    m, nl = xc.shape
    if nl != plan.n_locals[rank]:
        raise ValueError("decompose_sharded: X_local width does not match the plan")
    cap = max(1, min(int(d_max), plan.n_global))
    Y = torch.empty((cap, m), dtype=torch.float64, device=xc.device).t()
    T = torch.empty((cap, max(nl, 1)), dtype=torch.float64, device=xc.device)
    sel = np.zeros(cap, dtype=np.int64)
    hist = np.zeros(cap)
    res = Result()
    torch.cuda.current_stream(xc.device).synchronize()
    check(lib.rbd_decompose_sharded(ctx.handle, C.c_void_p(xc.data_ptr()), m, nl, ldx,
                                    plan.offsets[rank], plan.n_global, C.byref(cfg),
                                    C.c_void_p(Y.data_ptr()), C.c_void_p(T.data_ptr()),
                                    sel.ctypes.data_as(C.c_void_p), hist.ctypes.data_as(C.c_void_p),
                                    C.byref(res)))
    d = res.d
    return ShardedModel(Y[:, :d], T[:d, :nl], d, [int(s) for s in sel[:d]],
                        [float(h) for h in hist[:d]], res, plan, rank)


def assemble_T(T_local, plan: ShardPlan, group=None):
    """Gather every rank's d x n_local block into the global d x n T (all ranks)."""
    import torch
    import torch.distributed as dist
    d = T_local.shape[0]
    width = max(plan.n_locals)
    pad = torch.zeros((d, width), dtype=T_local.dtype, device=T_local.device)
    pad[:, : T_local.shape[1]] = T_local
    parts = [torch.empty_like(pad) for _ in range(plan.world)]
    dist.all_gather(parts, pad.contiguous(), group=group)
    return torch.cat([p[:, :nl] for p, nl in zip(parts, plan.n_locals)], dim=1)


def decompose_virtual(X, nranks: int, d_max: int, eps_r: float = 0.0,
                      n_locals: Optional[Sequence[int]] = None, ctx: Optional[Context] = None,
                      **cfg_kw):
    """Single-device emulation of the sharded loop (same kernels and payload
    protocol, exchange by device copies). Returns (Y_per_rank, T_global, d,
    selected, history, result)."""
    import torch
    lib = load_library()
    ctx = ctx or default_context(X.device.index or 0)
    cfg = make_config(d_max, eps_r, **cfg_kw)
    xc, ldx = _col_major_torch(X)
    m, n = xc.shape
    plan = plan_shards(n, nranks) if n_locals is None else ShardPlan(
        n, tuple(np.cumsum([0] + list(n_locals[:-1])).tolist()), tuple(n_locals))
    cap = max(1, min(int(d_max), n))
    shards = [xc[:, o:o + nl] for o, nl in zip(plan.offsets, plan.n_locals)]
    Ys = [torch.empty((cap, m), dtype=torch.float64, device=xc.device).t() for _ in range(nranks)]
    Ts = [torch.empty((cap, max(nl, 1)), dtype=torch.float64, device=xc.device)
          for nl in plan.n_locals]
    xp = (C.c_void_p * nranks)(*[C.c_void_p(s.data_ptr()) for s in shards])
    nlp = (C.c_int64 * nranks)(*plan.n_locals)
    yp = (C.c_void_p * nranks)(*[C.c_void_p(y.data_ptr()) for y in Ys])
    tp = (C.c_void_p * nranks)(*[C.c_void_p(t.data_ptr()) for t in Ts])
    sel = np.zeros(cap, dtype=np.int64)
    hist = np.zeros(cap)
    res = Result()
    torch.cuda.current_stream(xc.device).synchronize()
    check(lib.rbd_decompose_sharded_virtual(ctx.handle, nranks, xp, nlp, m, ldx, C.byref(cfg), yp,
                                            tp, sel.ctypes.data_as(C.c_void_p),
                                            hist.ctypes.data_as(C.c_void_p), C.byref(res)))
    d = res.d
    T = torch.cat([t[:d, :nl] for t, nl in zip(Ts, plan.n_locals)], dim=1)
    return [y[:, :d] for y in Ys], T, d, [int(s) for s in sel[:d]], [float(h) for h in hist[:d]], res
