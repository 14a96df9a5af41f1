"""A/B of two builds of librbd_b200.so on one workload: alternating decompose
calls through the bare C ABI (rbd_decompose_device), loop_ms medians.
Usage: tools/ab_lib.py WORKLOAD LIB_A LIB_B [reps] [d_max] [--f32|--diag]"""
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
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
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
d_max = int(sys.argv[5]) if len(sys.argv) > 5 else w.d_max
m, n = X.shape
libs = {}
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
    libs[tag] = (L, h)
cfg = Config()
libs["A"][0].rbd_config_default(C.byref(cfg))
cfg.d_max = d_max
cfg.eps_R = eps
Y = torch.empty((d_max, m), dtype=torch.float64, device="cuda").t()
T = torch.empty((d_max, n), dtype=torch.float64, device="cuda")
sel = np.zeros(d_max, dtype=np.int64)
hist = np.zeros(d_max)
out = {"A": [], "B": []}
sels = {}
for it in range(reps + 1):
    for tag, (L, h) in libs.items():
        r = Result()
        rc = (lambda *q: L.rbd_decompose_diag_device(*q[:6], C.c_void_p(DG.data_ptr()), m, *q[6:]) if DIAG
                  else (L.rbd_decompose_device_f32 if F32 else L.rbd_decompose_device)(*q))(h, C.c_void_p(X.data_ptr()), m, n, X.stride(1), C.byref(cfg),
                                    C.c_void_p(Y.data_ptr()), C.c_void_p(T.data_ptr()),
                                    sel.ctypes.data_as(C.c_void_p), hist.ctypes.data_as(C.c_void_p),
                                    C.byref(r))
        assert rc == 0, rc
        if it:
            out[tag].append(r.loop_ms)
        sels[tag] = sel[:r.d].copy()
xb = m * n * (4 if F32 else 8)
for tag in ("A", "B"):
    ms = float(np.median(out[tag]))
    print(f"{name} {tag} ({os.path.basename(sys.argv[2 if tag == 'A' else 3])}): loop {ms:9.3f} ms "
          f"{xb * d_max / ms / 1e6:8.1f} GB/s  runs {np.round(out[tag], 2)}")
print("same selections:", np.array_equal(sels["A"], sels["B"]))
