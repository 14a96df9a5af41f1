"""Two launches of K5 (fp64 DMMA projection) on one C4 batch, for ncu:
Y 65 536 x 512, X_new 65 536 x 16 384, T_new only (with_error=0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402

m, d, N = 65536, 512, 16384
g = torch.Generator(device="cuda").manual_seed(4)
Y = torch.randn(d, m, dtype=torch.float64, device="cuda", generator=g).t()
X = torch.randn(N, m, dtype=torch.float64, device="cuda", generator=g).t()
for _ in range(2):
    Tn, _err = rbd.project_batch(Y, X, with_error=False)
torch.cuda.synchronize()
print("ok", float(Tn[0, 0]))
