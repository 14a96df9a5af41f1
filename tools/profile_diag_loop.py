"""Run only the weighted C1 loop (bench_diag.py's weight), for traces / ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402

w = configs.WORKLOADS["C1-image-like"]
X = configs.c1_matrix(n=w.n, seed=w.seed, device="cuda")
m = X.shape[0]
eps = configs.eps_for(w, float(X.norm(dim=0).max()))
h, wd = configs.FRAME
yy, xx = np.meshgrid(np.linspace(-1, 1, h), np.linspace(-1, 1, wd), indexing="ij")
diag = (0.5 + 2.0 * np.exp(-(xx ** 2 + yy ** 2) / 0.3)).reshape(-1, order="F")[:m]
dg = torch.from_numpy(np.ascontiguousarray(diag, dtype=np.float64)).cuda()
ctx = rbd.Context(0)
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    g = rbd.decompose(X, d_max=w.d_max, eps_r=eps, diag=dg, ctx=ctx)
    print(f"run {it}: d={g.d} loop_ms={g.result.loop_ms:.2f} launches={g.result.launches}", flush=True)
