"""Run one workload's decomposition (warm-up + one measured call) for ncu
captures of the persistent loop kernel. Usage:
tools/profile_loop.py WORKLOAD [d_max] [f64|f32|diag]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1-image-like"
dmax = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
mode = sys.argv[3] if len(sys.argv) > 3 else "f64"
w, X, eps = bench.make_workload(name, torch.device("cuda:0"))
diag = None
if mode == "f32":     # fp32 storage mode
    X = X.float()
elif mode == "diag":  # row f1: bench_diag.py's pixel-importance weight (C1 frames)
    import numpy as np
    h, wd = configs.FRAME
    yy, xx = np.meshgrid(np.linspace(-1, 1, h), np.linspace(-1, 1, wd), indexing="ij")
    mask = 0.5 + 2.0 * np.exp(-(xx ** 2 + yy ** 2) / 0.3)
    diag = torch.from_numpy(mask.reshape(-1, order="F")[:X.shape[0]].astype(np.float64)).cuda()
ctx = rbd.Context(0)
for it in range(2):
    t = time.perf_counter()
    g = rbd.decompose(X, d_max=dmax or w.d_max, eps_r=eps, ctx=ctx, diag=diag)
    print(f"run {it}: d={g.d} loop_ms={g.result.loop_ms:.2f} init_ms={g.result.init_ms:.2f} "
          f"launches={g.result.launches} wall={time.perf_counter() - t:.3f}s", flush=True)
    del g
