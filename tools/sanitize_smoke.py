"""Small invocations of every kernel family in one process (a broad smoke run;
compute-sanitizer is not available on this pool): decompose (persistent loop, odd and even shapes,
reorth), diagonal weight, sharded virtual ranks, workspace, projection fp64 and
fp32 (tcgen05), compress, classify, container."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402
from paper_1503_05947_b200 import distributed  # noqa: E402

rng = np.random.default_rng(0)
for (m, n, d) in [(300, 40, 12), (4097, 33, 20), (33, 5, 5)]:
    x = rng.standard_normal((m, n))
    g = rbd.decompose(x, d_max=d)
    rbd.decompose(x.astype(np.float32), d_max=d)            # fp32 storage mode
    rbd.decompose_many([x, x[:, ::-1]], d_max=d)             # pipelined host entry
    rbd.decompose(x, d_max=d, reorthogonalize=True)
    rbd.decompose(x, d_max=d, diag=rng.uniform(0.5, 2.0, m))
    g.compress()
    g.project(x[:, 0])
    clf = rbd.Classifier(g, [str(j) for j in range(n)])
    clf.predict_batch(x[:, :7])
    with tempfile.TemporaryDirectory() as t:
        g.save(os.path.join(t, "m.rbd"), 0.0)
        rbd.load(os.path.join(t, "m.rbd"), device="cuda")
xd = torch.from_numpy(np.asfortranarray(rng.standard_normal((512, 64)))).cuda()
distributed.decompose_virtual(xd, 3, d_max=16)
ws = rbd.Workspace(torch.from_numpy(np.asfortranarray(rng.standard_normal((200, 30)))).cuda(), cap=8)
Y = torch.linalg.qr(torch.randn(1024, 128, device="cuda"))[0].float().t().contiguous().t()
X = torch.randn(256, 1024, device="cuda", dtype=torch.float32).t()
rbd.project_batch_f32(Y, X)
# CTA-pair kernel (d > 128 and N > 128), partial pair tiles in both
Y2 = torch.linalg.qr(torch.randn(1024, 300, device="cuda"))[0].float().t().contiguous().t()
X2 = torch.randn(300, 1024, device="cuda", dtype=torch.float32).t()
rbd.project_batch_f32(Y2, X2)
torch.cuda.synchronize()
print("sanitize smoke ok")
