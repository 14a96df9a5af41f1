"""One launch (after a warm-up) of a chosen secondary kernel, for ncu captures:
  tf32x3   K6 fp32 projection, C4 batch (Y 65 536 x 512, 16 384 new columns)
  compress compress_matrix of C1's model (k_compress_dmma)
  nearest  nearest-column step of the batched classify (C1 model, 16 384 queries)
  diag     one diagonal-weight decompose of C1's matrix, d = 40 (k_sweep_diag etc.)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402
from paper_1503_05947_b200._lib import check, load_library  # noqa: E402

op = sys.argv[1]
lib = load_library()
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
if op == "tf32x3":
    m, d, N = 65536, 512, 16384
    Y = torch.linalg.qr(torch.randn(m, d, device="cuda"))[0].float().t().contiguous().t()
    X = torch.randn(N, m, device="cuda", dtype=torch.float32).t()
    for _ in range(2):
        rbd.project_batch_f32(Y, X)
    torch.cuda.synchronize()
else:
    w = configs.WORKLOADS["C1-image-like"]
    X = configs.c1_matrix(n=w.n, seed=w.seed, device="cuda")
    eps = configs.eps_for(w, float(X.norm(dim=0).max()))
    if op == "diag":
        dg = torch.from_numpy(0.5 + 2.0 * np.random.default_rng(0).random(X.shape[0])).cuda()
        for _ in range(2):
            rbd.decompose(X, d_max=40, diag=dg)
    else:
        model = rbd.decompose(X, d_max=w.d_max, eps_r=eps)
        if op == "compress":
            for _ in range(2):
                model.compress()
        elif op == "nearest":
            clf = rbd.Classifier(model, [str(j) for j in range(X.shape[1])])
            nq = 16384
            g = torch.Generator(device="cuda").manual_seed(11)
            src = torch.randint(0, X.shape[1], (nq,), generator=g, device="cuda")
            Q = (X[:, src] + torch.randn(X.shape[0], nq, generator=g, device="cuda",
                                         dtype=torch.float64)).t().contiguous().t()
            for _ in range(2):
                clf.predict_indices(Q)
    torch.cuda.synchronize()
print("ok", op)
