"""A/B of a K5 knob (default RBD_K5_TILE; argv[3] names another, e.g. RBD_K5_TMA) on one C4 batch (Y 65 536 x 512,
X_new 65 536 x 16 384, fp64): alternating runs, CUDA events, plus a bitwise
comparison of T_new and the error indicator across the shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402

m, d, N = 65536, 512, 16384
g = torch.Generator(device="cuda").manual_seed(4)
Y = torch.linalg.qr(torch.randn(m, d, dtype=torch.float64, device="cuda", generator=g))[0]
Y = Y.t().contiguous().t()
X = torch.randn(N, m, dtype=torch.float64, device="cuda", generator=g).t()
tiles = sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "1"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
var = sys.argv[3] if len(sys.argv) > 3 else "RBD_K5_TILE"
ctx = rbd.Context(0)
st = torch.cuda.ExternalStream(ctx.stream)
res = {t: [] for t in tiles}
outs = {}
for it in range(reps + 1):
    for t in tiles:
        os.environ[var] = t
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        Tn, err = rbd.project_batch(Y, X, ctx=ctx)
        e1.record(st)
        torch.cuda.synchronize()
        if it:
            res[t].append(e0.elapsed_time(e1))
        outs[t] = (Tn.cpu().numpy(), err.cpu().numpy())
flops = 2.0 * m * d * N
for t, v in res.items():
    ms = float(np.median(v))
    print(f"{var}={t}: {ms:.2f} ms  {flops / ms / 1e9:.1f} TFLOP/s  runs {np.round(v, 2)}")
a = outs[tiles[0]]
for t in tiles[1:]:
    print(f"{var}={t} bitwise equal to {var}={tiles[0]}: T {np.array_equal(a[0], outs[t][0])} "
          f"err {np.array_equal(a[1], outs[t][1])}")
Yt = Y.t().contiguous()
ref = Yt @ X
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    ref = Yt @ X
e1.record()
torch.cuda.synchronize()
print(f"cuBLAS DGEMM: {e0.elapsed_time(e1) / 3:.2f} ms  {flops / (e0.elapsed_time(e1) / 3) / 1e9:.1f} TFLOP/s")
