"""Row f4 measurement: batched Classifier::predict with a classifier fitted on C1's
matrix (32 256 x 2 432 training columns, d = 400) and 16 384 device-resident
queries (training columns + noise); CUDA-event times of the whole batched call
(rbd_classify_batch), of its projection (K5) and of the nearest-column kernel;
the oracle (classify.cpp restated) on a bounded query sample. Prints one JSON line."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402
from paper_1503_05947_b200._lib import check, load_library  # noqa: E402
import oracle  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
w = configs.WORKLOADS["C1-image-like"]
X = configs.c1_matrix(n=w.n, seed=w.seed, device="cuda")
m, n = X.shape
eps = configs.eps_for(w, float(X.norm(dim=0).max()))
clf = rbd.fit(X, [str(j) for j in range(n)], d_max=w.d_max, eps_r=eps)
d = clf.model.d
g = torch.Generator(device="cuda").manual_seed(11)
src = torch.randint(0, n, (nq,), generator=g, device="cuda")
Q = X[:, src] + 2.0 * torch.randn(m, nq, generator=g, device="cuda", dtype=torch.float64)
Q = Q.t().contiguous().t()
Yd, Td = clf._device_model()
ctx = clf.model._ctx
lib = load_library()
best = torch.empty(nq, dtype=torch.int64, device="cuda")
coords = torch.empty((nq, d), dtype=torch.float64, device="cuda")
stream = torch.cuda.ExternalStream(ctx.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, reps=10):
    fn()
    ctx.synchronize()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
t_all = timed(lambda: check(lib.rbd_classify_batch(ctx.handle, p(Yd), m, d, Yd.stride(1), p(Td), n,
                                                   p(Q), nq, Q.stride(1), p(best), None)))
t_proj = timed(lambda: check(lib.rbd_project_batch(ctx.handle, p(Yd), m, d, Yd.stride(1), p(Q), nq,
                                                   Q.stride(1), p(coords), None)))
t_nn = timed(lambda: check(lib.rbd_nearest_columns(ctx.handle, p(coords), d, nq, d, p(Td), n,
                                                   p(best), None)))
hits = float((best == src).double().mean())
# oracle on a bounded sample
k = 64
Yh, Th, Qh = Yd.cpu().numpy(), Td.cpu().numpy(), Q[:, :k].cpu().numpy()
t0 = time.perf_counter()
rb, _ = oracle.predict_batch(Yh, Th, Qh, nthreads=1)
t1 = time.perf_counter() - t0
nn_flops = 3.0 * d * n * nq
print(json.dumps({
    "row": "f4 batched classify", "train": f"C1 ({m}x{n}), d={d}", "queries": nq,
    "queries_per_s": nq / (t_all / 1e3), "ms_per_batch": t_all,
    "projection_ms": t_proj, "projection_tflops": 2.0 * m * d * nq / (t_proj / 1e3) / 1e12,
    "nearest_ms": t_nn, "nearest_tflops": nn_flops / (t_nn / 1e3) / 1e12,
    "nearest_flops_note": "3 flops per (coordinate, column, query): subtract + fma",
    "fp64_reference_rate_tflops": 36.2,
    "fp64_reference_note": "cuBLAS DGEMM on the K5 shape, measured on this pool (DESIGN §4)",
    "own_column_hits": hits,
    "oracle_single_thread": {"queries": k, "seconds": t1, "queries_per_s": k / t1,
                             "agree_on_sample": bool(np.array_equal(rb, best[:k].cpu().numpy()))},
}))
