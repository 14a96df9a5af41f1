"""Row f2 measurement: write and read the RBD1 container of C1's model (Y 32 256 x 400,
T 400 x 2 432: 111 MB) between HBM and a file (page cache under /tmp), through the
C ABI; the oracle's writer (numpy byte restatement of io.cpp) on host copies beside
it. Prints one JSON line."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402
import oracle  # noqa: E402

w = configs.WORKLOADS["C1-image-like"]
X = configs.c1_matrix(n=w.n, seed=w.seed, device="cuda")
eps = configs.eps_for(w, float(X.norm(dim=0).max()))
model = rbd.decompose(X, d_max=w.d_max, eps_r=eps)
m, n, d = X.shape[0], X.shape[1], model.d
nbytes = 29 + 8 * (m * d + d * n + 1 + d)
base = sys.argv[1] if len(sys.argv) > 1 else None
path = os.path.join(tempfile.mkdtemp(dir=base), "c1.rbd")
reps = 5
model.save(path, eps)
t0 = time.perf_counter()
for _ in range(reps):
    model.save(path, eps)
tw = (time.perf_counter() - t0) / reps
rbd.load(path, device="cuda")
t0 = time.perf_counter()
for _ in range(reps):
    back, _ = rbd.load(path, device="cuda")
torch.cuda.synchronize()
tr = (time.perf_counter() - t0) / reps
Yh, Th = model.Y.cpu().numpy(), model.T.cpu().numpy()
t0 = time.perf_counter()
for _ in range(reps):
    with open(path + ".oracle", "wb") as f:
        f.write(oracle.model_bytes(Yh, Th, eps, model.residual_history, 0))
to = (time.perf_counter() - t0) / reps
same = open(path, "rb").read() == open(path + ".oracle", "rb").read()
print(json.dumps({"row": "f2 model container", "dir": os.path.dirname(path), "model": f"C1 ({m}x{d} Y, {d}x{n} T)",
                  "bytes": nbytes, "write_hbm_to_file_gbs": nbytes / tw / 1e9,
                  "read_file_to_hbm_gbs": nbytes / tr / 1e9, "write_ms": tw * 1e3,
                  "read_ms": tr * 1e3, "oracle_host_write_gbs": nbytes / to / 1e9,
                  "bytes_equal_oracle": same, "exact_round_trip": bool(torch.equal(back.Y, model.Y))}))
