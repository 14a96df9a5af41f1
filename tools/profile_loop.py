"""Run the C1 decomposition (warm-up + one measured call) for ncu launch lists."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1-image-like"
dmax = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = configs.WORKLOADS[name]
X = configs.c1_matrix(n=w.n, seed=w.seed, device="cuda")
eps = configs.eps_for(w, float(X.norm(dim=0).max()))
if len(sys.argv) > 3 and sys.argv[3] == "f32":   # fp32 storage mode
    X = X.float()
ctx = rbd.Context(0)
for it in range(2):
    t = time.perf_counter()
    g = rbd.decompose(X, d_max=dmax or w.d_max, eps_r=eps, ctx=ctx)
    print(f"run {it}: d={g.d} loop_ms={g.result.loop_ms:.2f} init_ms={g.result.init_ms:.2f} "
          f"launches={g.result.launches} wall={time.perf_counter() - t:.3f}s", flush=True)
