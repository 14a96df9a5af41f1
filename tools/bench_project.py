"""C4 out-of-sample compression: RBD on the 65536 x 8192 rank-512 stage, then
project 16 batches of 16384 new columns (T_new = Y'X_new, err = ||x||^2-||t||^2).
Times rbd_project_batch (our kernels) and, for context, cuBLAS DGEMM via torch."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    w = configs.C4
    nb = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    batch = 16384
    g = torch.Generator(device=dev)
    g.manual_seed(w.seed)
    m, rank = w.m, 512
    U = torch.linalg.qr(torch.randn(m, rank, dtype=torch.float64, device=dev, generator=g))[0]
    s = torch.as_tensor(configs.spectrum("C4", rank), device=dev)
    V = torch.linalg.qr(torch.randn(w.n, rank, dtype=torch.float64, device=dev, generator=g))[0]
    X = ((V * s) @ U.t()).t() + 1e-3 * torch.randn(m, w.n, dtype=torch.float64, device=dev, generator=g)
    X = X.t().contiguous().t()
    ctx = rbd.Context(0)
    t0 = time.time()
    mdl = rbd.decompose(X, d_max=512, ctx=ctx)
    print(f"[rbd stage] d={mdl.d} loop {mdl.result.loop_ms:.1f} ms ({time.time() - t0:.1f}s wall)")
    Y = mdl.Y.t().contiguous().t()
    d = mdl.d
    flops = 2.0 * m * d * batch
    batches = []
    for b in range(nb):
        coef = torch.randn(rank, batch, dtype=torch.float64, device=dev, generator=g) / np.sqrt(w.n)
        Xn = (U * s) @ coef + 1e-3 * torch.randn(m, batch, dtype=torch.float64, device=dev, generator=g)
        batches.append(Xn.t().contiguous().t())
    torch.cuda.synchronize()
    # ours
    rbd.project_batch(Y, batches[0], ctx=ctx)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.ExternalStream(ctx.stream, device=dev)
    e0.record(st)
    for Xn in batches:
        Tn, err = rbd.project_batch(Y, Xn, ctx=ctx)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / nb
    print(f"[ours] {ms:.2f} ms/batch -> {flops / ms / 1e9:.2f} TFLOP/s (fp64, incl. error indicator)")
    e0.record(st)
    for Xn in batches:
        Tn2, _ = rbd.project_batch(Y, Xn, with_error=False, ctx=ctx)
    e1.record(st)
    torch.cuda.synchronize()
    ms2 = e0.elapsed_time(e1) / nb
    print(f"[ours, T only] {ms2:.2f} ms/batch -> {flops / ms2 / 1e9:.2f} TFLOP/s")
    # fp32 mode: tcgen05 kind::tf32 with the 3xTF32 split
    Y32 = Y.to(torch.float32).t().contiguous().t()
    b32 = [Xn.to(torch.float32).t().contiguous().t() for Xn in batches]
    rbd.project_batch_f32(Y32, b32[0], ctx=ctx)
    torch.cuda.synchronize()
    e0.record(st)
    for Xn in b32:
        T32, err32 = rbd.project_batch_f32(Y32, Xn, ctx=ctx)
    e1.record(st)
    torch.cuda.synchronize()
    ms3 = e0.elapsed_time(e1) / nb
    print(f"[ours fp32 tcgen05 3xTF32] {ms3:.2f} ms/batch -> {flops / ms3 / 1e9:.2f} TFLOP/s "
          f"(fp32-equivalent; 3 tf32 MMAs per product)")
    Yt32 = Y32.t().contiguous()
    torch.backends.cuda.matmul.allow_tf32 = False
    e0.record()
    for Xn in b32:
        Tc32 = torch.matmul(Yt32, Xn)
    e1.record()
    torch.cuda.synchronize()
    ms4 = e0.elapsed_time(e1) / nb
    print(f"[cuBLAS SGEMM fp32] {ms4:.2f} ms/batch -> {flops / ms4 / 1e9:.2f} TFLOP/s")
    ref32 = Y32.double().t() @ b32[-1].double()
    sc32 = (b32[-1].double() ** 2).sum(0).sqrt()
    print(f"[check fp32] max|dT|/||x|| = {float(((T32.double() - ref32).abs() / sc32).max()):.2e}")
    # cuBLAS DGEMM (context / ceiling)
    Yt = Y.t().contiguous()
    torch.matmul(Yt, batches[0])
    torch.cuda.synchronize()
    e0.record()
    for Xn in batches:
        Tc = torch.matmul(Yt, Xn)
    e1.record()
    torch.cuda.synchronize()
    msc = e0.elapsed_time(e1) / nb
    print(f"[cuBLAS DGEMM] {msc:.2f} ms/batch -> {flops / msc / 1e9:.2f} TFLOP/s")
    err_ref = (batches[-1] * batches[-1]).sum(0) - (Tc * Tc).sum(0)
    scale = (batches[-1] * batches[-1]).sum(0)
    print(f"[check] max|dT|/||x|| = {float(((Tn - Tc).abs() / scale.sqrt()).max()):.2e}, "
          f"max|derr|/||x||^2 = {float(((err - err_ref.clamp(min=0)).abs() / scale).max()):.2e}")


if __name__ == "__main__":
    main()
