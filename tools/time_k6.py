"""Device timing of K6 (fp32 out-of-sample compression, 3xTF32 on tcgen05) on the
C4 batch shape (m = 65536, d = 512, N = 16384). RBD_K6_PAIR / RBD_K6_SPLITK pick
the kernel and the split. Usage: tools/time_k6.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
dev = torch.device("cuda:0")
m, d, N = 65536, 512, 16384
g = torch.Generator(device=dev)
g.manual_seed(4)
Y = torch.linalg.qr(torch.randn(m, d, dtype=torch.float32, device=dev, generator=g))[0].t().contiguous().t()
X = torch.randn(N, m, dtype=torch.float32, device=dev, generator=g).t()
ctx = rbd.Context(0)
st = torch.cuda.ExternalStream(ctx.stream, device=dev)
for with_error in (True, False):
    rbd.project_batch_f32(Y, X, with_error=with_error, ctx=ctx)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        T, err = rbd.project_batch_f32(Y, X, with_error=with_error, ctx=ctx)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"K6 pair={os.environ.get('RBD_K6_PAIR', 'auto')} splitk={os.environ.get('RBD_K6_SPLITK', 'auto')} "
          f"with_error={with_error}: {ms:.3f} ms/batch -> {2.0 * m * d * N / ms / 1e9:.1f} TFLOP/s fp32-equivalent "
          f"({3 * 2.0 * m * d * N / ms / 1e9:.0f} TFLOP/s of kind::tf32 MMA)", flush=True)
ref = (Y.double().t() @ X[:, :256].double())
print("max |dT| / ||x|| vs fp64 on 256 columns:",
      float(((T[:, :256].double() - ref).abs() / X[:, :256].double().norm(dim=0)).max()))
