"""One diagonal-weight decompose of C1's matrix (d_max from argv, default 60) after
one warm-up, for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 60
w = configs.WORKLOADS["C1-image-like"]
X = configs.c1_matrix(n=w.n, seed=w.seed, device="cuda")
m = X.shape[0]
dg = torch.from_numpy(0.5 + 2.0 * np.random.default_rng(0).random(m)).cuda()
for it in range(2):
    g = rbd.decompose(X, d_max=d, diag=dg)
    print(f"run {it}: d={g.d} loop_ms={g.result.loop_ms:.2f} launches={g.result.launches}", flush=True)
