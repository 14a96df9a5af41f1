"""A/B of env-knob combinations of the persistent loop on one workload, arms
alternated in one process (clock drift hits every arm alike), then one
RBD_PHASE_TIMING run per arm (CTA 0 phase split, stderr; needs a library
built with RBD_NVCC_DEFS=-DRBD_INSTRUMENT=1).
Usage: tools/ab_arms.py WORKLOAD "A=1,B=2" "A=0" ... [--reps R] [--f32]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1503_05947_b200 as rbd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("arms", nargs="+")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--f32", action="store_true")
ap.add_argument("--phases", action="store_true")
args = ap.parse_args()


def parse(arm):
    return dict(kv.split("=", 1) for kv in arm.split(",") if kv)


w, X, eps = bench.make_workload(args.workload, torch.device("cuda:0"))
if args.f32:
    X = X.float()
ctx = rbd.Context(0)
res = {a: [] for a in args.arms}
sel = {}
for it in range(args.reps + 1):
    for arm in args.arms:
        env = parse(arm)
        os.environ.update(env)
        g = rbd.decompose(X, d_max=w.d_max, eps_r=eps, ctx=ctx)
        for k in env:
            del os.environ[k]
        if it:
            res[arm].append(g.result.loop_ms)
        sel[arm] = g.selected
        del g
xb = w.m * w.n * (4 if args.f32 else 8)
for arm, r in res.items():
    ms = float(np.median(r))
    print(f"{args.workload} [{arm:>30s}]: loop {ms:9.3f} ms  {xb * w.d_max / ms / 1e6:8.1f} GB/s  runs {np.round(r, 2)}",
          flush=True)
print("same selections:", all(sel[a] == sel[args.arms[0]] for a in args.arms), flush=True)
if args.phases:
    for arm in args.arms:
        env = parse(arm)
        os.environ.update(env)
        os.environ["RBD_PHASE_TIMING"] = "1"
        print(f"--- phases [{arm}]", flush=True)
        sys.stderr.flush()
        g = rbd.decompose(X, d_max=w.d_max, eps_r=eps, ctx=ctx)
        torch.cuda.synchronize()
        sys.stderr.flush()
        del g
        for k in list(env) + ["RBD_PHASE_TIMING"]:
            del os.environ[k]
