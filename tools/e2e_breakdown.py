"""Where the end-to-end (host buffer) decompose time goes on C1: pinned H2D of X,
the device-resident decompose, and the host entry as a whole."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402

w = configs.WORKLOADS["C1-image-like"]
Xd = configs.c1_matrix(n=w.n, seed=w.seed, device="cuda")
m, n = Xd.shape
eps = configs.eps_for(w, float(Xd.norm(dim=0).max()))
ctx = rbd.Context(0)
Xh_t = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
Xh_t.copy_(Xd.t())
Xh = Xh_t.numpy().T
dst = torch.empty_like(Xh_t, device="cuda")
for it in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    dst.copy_(Xh_t, non_blocking=True)
    torch.cuda.synchronize()
    h2d = time.perf_counter() - t
    t = time.perf_counter()
    g = rbd.decompose(Xd, d_max=w.d_max, eps_r=eps, ctx=ctx)
    torch.cuda.synchronize()
    dev = time.perf_counter() - t
    t = time.perf_counter()
    g2 = rbd.decompose(Xh, d_max=w.d_max, eps_r=eps, ctx=ctx)
    host = time.perf_counter() - t
    print(f"it {it}: H2D {h2d*1e3:.2f} ms ({m*n*8/h2d/1e9:.1f} GB/s)  device decompose {dev*1e3:.2f} ms "
          f"(loop {g.result.loop_ms:.2f})  host decompose {host*1e3:.2f} ms (loop {g2.result.loop_ms:.2f}, "
          f"init {g2.result.init_ms:.2f})", flush=True)
