"""Stress of the K6 CTA-pair kernel: random shapes against the single-CTA kernel
at equal split-K (bitwise), and the C4 batch shape run to run (bitwise).
Usage: tools/stress_k6.py [iterations]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_05947_b200 as rbd  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
dev = torch.device("cuda:0")
rng = np.random.default_rng(11)
g = torch.Generator(device=dev)
g.manual_seed(1)
bad = 0
for it in range(iters):
    m = int(rng.integers(33, 20000))
    d = int(rng.integers(129, 700))
    N = int(rng.integers(129, 1500))
    sk = int(rng.integers(1, 5))
    mp = (m + 3) // 4 * 4
    Y = torch.randn(d, mp, dtype=torch.float32, device=dev, generator=g).t()[:m]
    X = torch.randn(N, mp, dtype=torch.float32, device=dev, generator=g).t()[:m]
    os.environ["RBD_K6_SPLITK"] = str(sk)
    os.environ["RBD_K6_PAIR"] = "0"
    T1, e1 = rbd.project_batch_f32(Y, X)
    os.environ["RBD_K6_PAIR"] = "1"
    T2, e2 = rbd.project_batch_f32(Y, X)
    torch.cuda.synchronize()
    if not (torch.equal(T1, T2) and torch.equal(e1, e2)):
        bad += 1
        print("MISMATCH", m, d, N, sk, float((T1 - T2).abs().max()), flush=True)
print(f"random shapes: {iters} cases, {bad} mismatches", flush=True)
del os.environ["RBD_K6_SPLITK"], os.environ["RBD_K6_PAIR"]
m, d, N = 65536, 512, 16384
Y = torch.linalg.qr(torch.randn(m, d, dtype=torch.float32, device=dev, generator=g))[0].t().contiguous().t()
X = torch.randn(N, m, dtype=torch.float32, device=dev, generator=g).t()
T0, e0 = rbd.project_batch_f32(Y, X)
T0, e0 = T0.clone(), e0.clone()
rep_bad = 0
for it in range(40):
    T, e = rbd.project_batch_f32(Y, X)
    torch.cuda.synchronize()
    if not (torch.equal(T, T0) and torch.equal(e, e0)):
        rep_bad += 1
print(f"C4 batch run to run: 40 repeats, {rep_bad} differing", flush=True)
sys.exit(1 if (bad or rep_bad) else 0)
