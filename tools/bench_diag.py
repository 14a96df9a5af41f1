"""Row f1 measurement: the diagonal-weight greedy loop on C1's matrix (32 256 x 2 432,
d_max 400, C1's stop rule) with a smooth pixel-importance weight, timed with the
library's CUDA events; the identity loop on the same matrix beside it, and the
oracle (single thread, restating the reference's O(n d^2)-per-step error scan)
on a bounded sample of steps. Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = configs.WORKLOADS["C1-image-like"]
X = configs.c1_matrix(n=w.n, seed=w.seed, device="cuda")
m, n = X.shape
eps = configs.eps_for(w, float(X.norm(dim=0).max()))
# weight: a centred Gaussian importance mask over the 192 x 168 frame, in [0.5, 2.5]
h, wd = configs.FRAME
yy, xx = np.meshgrid(np.linspace(-1, 1, h), np.linspace(-1, 1, wd), indexing="ij")
mask = 0.5 + 2.0 * np.exp(-(xx ** 2 + yy ** 2) / 0.3)
diag = mask.reshape(-1, order="F")[:m].astype(np.float64)
dg = torch.from_numpy(diag).cuda()
ctx = rbd.Context(0)
for _ in range(2):
    g = rbd.decompose(X, d_max=w.d_max, eps_r=eps, diag=dg, ctx=ctx)
    gi = rbd.decompose(X, d_max=w.d_max, eps_r=eps, ctx=ctx)
lw, li, dw, di = [], [], [], []
for _ in range(steps):
    g = rbd.decompose(X, d_max=w.d_max, eps_r=eps, diag=dg, ctx=ctx)
    lw.append(g.result.loop_ms)
    dw.append(g.d)
    gi = rbd.decompose(X, d_max=w.d_max, eps_r=eps, ctx=ctx)
    li.append(gi.result.loop_ms)
    di.append(gi.d)
bytes_step = m * n * 8
val_w = bytes_step * np.mean(dw) / (np.mean(lw) / 1e3) / 1e9
val_i = bytes_step * np.mean(di) / (np.mean(li) / 1e3) / 1e9
# oracle sample (single thread; the reference's scan is O(n d^2) per step)
import oracle  # noqa: E402

Xh = np.asfortranarray(X.cpu().numpy())
k_or = 24
t0 = time.perf_counter()
r = oracle.decompose(Xh, w.d_max, eps, diag=diag, max_steps=k_or)
dt = time.perf_counter() - t0
agree = r.selected == g.selected[:k_or]
print(json.dumps({
    "row": "f1 diagonal weight", "workload": "C1-image-like + Gaussian pixel weight [0.5, 2.5]",
    "m": m, "n": n, "d_max": w.d_max, "d_reached": int(np.mean(dw)),
    "loop_ms": float(np.mean(lw)), "ms_per_greedy_step": float(np.mean(lw)) / np.mean(dw),
    "effective_gbs": val_w, "identity_loop_ms": float(np.mean(li)), "identity_gbs": val_i,
    "launches_per_decompose": g.result.launches,
    "oracle_single_thread": {"steps": r.d, "seconds": dt,
                             "effective_gbs": bytes_step * r.d / dt / 1e9,
                             "selected_prefix_equal": bool(agree)},
}), flush=True)
