"""A/B of a per-launch environment knob of the persistent loop (e.g.
RBD_YDELAY) on one workload, alternating values in one process so clock
drift hits every arm alike. Usage: tools/ab_env.py WORKLOAD VAR v1,v2,... [reps] [f32]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1503_05947_b200 as rbd  # noqa: E402

name, var, vals = sys.argv[1], sys.argv[2], sys.argv[3].split(",")
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
f32 = len(sys.argv) > 5 and sys.argv[5] == "f32"
w, X, eps = bench.make_workload(name, torch.device("cuda:0"))
if f32:
    X = X.float()
ctx = rbd.Context(0)
res = {v: [] for v in vals}
sel = {}
for it in range(reps + 1):
    for v in vals:
        os.environ[var] = v
        g = rbd.decompose(X, d_max=w.d_max, eps_r=eps, ctx=ctx)
        if it:
            res[v].append(g.result.loop_ms)
        sel[v] = g.selected
        del g
xb = w.m * w.n * (4 if f32 else 8)
for v, r in res.items():
    ms = float(np.median(r))
    print(f"{name}{' f32' if f32 else ''} {var}={v:>6s}: loop {ms:9.3f} ms  {xb * w.d_max / ms / 1e6:8.1f} GB/s  "
          f"runs {np.round(r, 2)}")
print("same selections:", all(sel[v] == sel[vals[0]] for v in vals))
