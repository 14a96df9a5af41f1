"""K5 timing on one C4 batch (Y 65 536 x 512, X_new 65 536 x 16 384, fp64):
best of 5, CUDA events; T_new only and with the error indicator."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402

m, d, N = 65536, 512, 16384
g = torch.Generator(device="cuda").manual_seed(4)
Y = torch.randn(d, m, dtype=torch.float64, device="cuda", generator=g).t()
X = torch.randn(N, m, dtype=torch.float64, device="cuda", generator=g).t()
ref = (Y.t() @ X)
for we in (False, True):
    best = 1e9
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        Tn, err = rbd.project_batch(Y, X, with_error=we)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    rel = float(((Tn - ref).abs().max() / ref.abs().max()))
    print(f"with_error={we}: {best:.2f} ms  {2 * m * d * N / best / 1e9:.1f} TFLOP/s  max rel diff vs cuBLAS {rel:.1e}")
