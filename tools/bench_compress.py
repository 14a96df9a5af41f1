"""Row f3 measurement: compress_matrix Y T for C1's model (32 256 x 400 times
400 x 2 432) on the FP64 tensor cores (rbd_compress_device), CUDA events, beside
cuBLAS DGEMM (torch.matmul in float64) on the same operands. Prints one JSON line."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402
from paper_1503_05947_b200._lib import check, load_library  # noqa: E402

w = configs.WORKLOADS["C1-image-like"]
X = configs.c1_matrix(n=w.n, seed=w.seed, device="cuda")
eps = configs.eps_for(w, float(X.norm(dim=0).max()))
model = rbd.decompose(X, d_max=w.d_max, eps_r=eps)
Y, T = model.Y, model.T.contiguous()
m, d = Y.shape
n = T.shape[1]
V = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
lib = load_library()
ctx = model._ctx
stream = torch.cuda.ExternalStream(ctx.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
run = lambda: check(lib.rbd_compress_device(ctx.handle, C.c_void_p(Y.data_ptr()), m, d,  # noqa: E731
                                            Y.stride(1), C.c_void_p(T.data_ptr()), n, n,
                                            C.c_void_p(V.data_ptr()), m))
run()
ctx.synchronize()
reps = 10
e0.record(stream)
for _ in range(reps):
    run()
e1.record(stream)
torch.cuda.synchronize()
t_ours = e0.elapsed_time(e1) / reps
Yc = Y.contiguous()
ref = Yc @ T
torch.cuda.synchronize()
e0.record()
for _ in range(reps):
    ref = Yc @ T
e1.record()
torch.cuda.synchronize()
t_cublas = e0.elapsed_time(e1) / reps
flops = 2.0 * m * d * n
err = float(((V - ref).abs() / (Y.abs() @ T.abs() * d * 2.2e-16 + 1e-300)).max())
print(json.dumps({"row": "f3 compress_matrix", "shape": f"{m}x{d} @ {d}x{n}",
                  "ours_ms": t_ours, "ours_tflops": flops / (t_ours / 1e3) / 1e12,
                  "cublas_dgemm_ms": t_cublas, "cublas_tflops": flops / (t_cublas / 1e3) / 1e12,
                  "max_err_over_dot_bound": err}))
