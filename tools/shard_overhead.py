"""Per-step cost of the sharded mode (step kernel, NCCL record allgather, pack,
NCCL payload allreduce, select; replayed from a CUDA graph, or eager with
RBD_SHARD_GRAPH=0) against the single-GPU persistent loop, on C1 (or the
workload named by argv[1]) at world 1 (NCCL with one rank). Prints one JSON line."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs, distributed as rd  # noqa: E402
from paper_1503_05947_b200._lib import check, load_library  # noqa: E402

import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1-image-like"
w, X, _ = bench.make_workload(name, torch.device("cuda"))
m, n = X.shape
ctx = rbd.Context(0)
buf = C.create_string_buffer(128)
check(load_library().rbd_comm_unique_id(buf))
rd.init_comm(ctx, 0, 1, bytes(buf.raw))
plan = rd.plan_shards(n, 1)
out = {}
def eager():
    os.environ["RBD_SHARD_GRAPH"] = "0"
    try:
        return rd.decompose_sharded(X, plan, 0, w.d_max, 0.0, ctx=ctx)
    finally:
        os.environ.pop("RBD_SHARD_GRAPH")


for name, fn in (("persistent", lambda: rbd.decompose(X, d_max=w.d_max, ctx=ctx)),
                 ("sharded_world1_graph", lambda: rd.decompose_sharded(X, plan, 0, w.d_max, 0.0,
                                                                       ctx=ctx)),
                 ("sharded_world1_eager", eager)):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.ExternalStream(ctx.stream)
    e0.record(st)
    r = fn()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out[name] = {"ms": ms, "d": r.d, "us_per_step": 1e3 * ms / r.d,
                 "gbs": m * n * 8 * r.d / (ms / 1e3) / 1e9}
print(json.dumps(out))
