"""Bitwise comparison of two builds of librbd_b200.so on one workload: Y, T,
selections and history of rbd_decompose_device (a change meant to keep the
arithmetic must give identical bytes). Usage: tools/bits_ab.py WORKLOAD LIB_A LIB_B [d_max] [--f32|--diag]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1503_05947_b200._lib import Config, Result  # noqa: E402

F32 = "--f32" in sys.argv
if F32:
    sys.argv.remove("--f32")
DIAG = "--diag" in sys.argv   # the weighted loop with tools/profile_diag_loop.py's weight
if DIAG:
    sys.argv.remove("--diag")
name, la, lb = sys.argv[1], sys.argv[2], sys.argv[3]
w, X, eps = bench.make_workload(name, torch.device("cuda:0"))
if F32:   # fp32 storage mode: the same values rounded to float32
    X = X.float()
if DIAG:
    from paper_1503_05947_b200 import configs
    hh, ww = configs.FRAME
    gy, gx = np.meshgrid(np.linspace(-1, 1, hh), np.linspace(-1, 1, ww), indexing="ij")
    dgn = (0.5 + 2.0 * np.exp(-(gx ** 2 + gy ** 2) / 0.3)).reshape(-1, order="F")
    dgn = np.resize(dgn, X.shape[0])
    DG = torch.from_numpy(np.ascontiguousarray(dgn, dtype=np.float64)).cuda()
d_max = int(sys.argv[4]) if len(sys.argv) > 4 else w.d_max
m, n = X.shape
outs = {}
for tag, path in (("A", la), ("B", lb)):
    L = C.CDLL(os.path.abspath(path))
    L.rbd_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    L.rbd_config_default.argtypes = [C.POINTER(Config)]
    for fn in ("rbd_decompose_device", "rbd_decompose_device_f32"):
        getattr(L, fn).argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                   C.POINTER(Config), C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.POINTER(Result)]
    L.rbd_decompose_diag_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                            C.POINTER(Config), C.c_void_p, C.c_int64, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(Result)]
    h = C.c_void_p()
    assert L.rbd_ctx_create(0, C.byref(h)) == 0
    cfg = Config()
    L.rbd_config_default(C.byref(cfg))
    cfg.d_max = d_max
    cfg.eps_R = eps
    Y = torch.empty((d_max, m), dtype=torch.float64, device="cuda").t()
    T = torch.empty((d_max, n), dtype=torch.float64, device="cuda")
    sel = np.zeros(d_max, dtype=np.int64)
    hist = np.zeros(d_max)
    r = Result()
    rc = (lambda *q: L.rbd_decompose_diag_device(*q[:6], C.c_void_p(DG.data_ptr()), m, *q[6:]) if DIAG
                  else (L.rbd_decompose_device_f32 if F32 else L.rbd_decompose_device)(*q))(h, C.c_void_p(X.data_ptr()), m, n, X.stride(1), C.byref(cfg),
                                C.c_void_p(Y.data_ptr()), C.c_void_p(T.data_ptr()),
                                sel.ctypes.data_as(C.c_void_p), hist.ctypes.data_as(C.c_void_p), C.byref(r))
    assert rc == 0, rc
    torch.cuda.synchronize()
    outs[tag] = (r.d, sel[:r.d].copy(), hist[:r.d].copy(), Y[:, :r.d].cpu().numpy().copy(),
                 T[:r.d].cpu().numpy().copy())
a, b = outs["A"], outs["B"]
same = (a[0] == b[0] and np.array_equal(a[1], b[1]) and a[2].tobytes() == b[2].tobytes()
        and a[3].tobytes() == b[3].tobytes() and a[4].tobytes() == b[4].tobytes())
print(f"{name} d={a[0]}/{b[0]} bitwise identical: {same}; max|dY| {np.abs(a[3] - b[3]).max() if a[3].shape == b[3].shape else 'shape'}")
