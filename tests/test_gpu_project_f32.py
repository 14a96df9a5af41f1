"""fp32 mode of the out-of-sample compression (tcgen05 kind::tf32, 3xTF32)
against fp64 on the same fp32-rounded inputs; north_star tolerance 1e-4
(relative to ||x_j||), with the 3xTF32 split expected to be far tighter."""
import numpy as np
import pytest

import oracle
import paper_1503_05947_b200 as rbd

pytestmark = pytest.mark.gpu


def run(cuda, m, d, N, seed=0):
    import torch
    g = torch.Generator(device=cuda)
    g.manual_seed(seed)
    Y = torch.linalg.qr(torch.randn(m, d, dtype=torch.float64, device=cuda, generator=g))[0]
    Xn = torch.randn(m, N, dtype=torch.float64, device=cuda, generator=g)
    Y32 = Y.to(torch.float32).t().contiguous().t()
    X32 = Xn.to(torch.float32).t().contiguous().t()
    Tn, err = rbd.project_batch_f32(Y32, X32)
    Y64, X64 = Y32.double(), X32.double()
    Tr = Y64.t() @ X64
    xx = (X64 * X64).sum(0)
    er = (xx - (Tr * Tr).sum(0)).clamp(min=0)
    scale = xx.sqrt()
    dT = float(((Tn.double() - Tr).abs() / scale).max())
    dE = float(((err - er).abs() / xx).max())
    return dT, dE


@pytest.mark.parametrize("m,d,N", [(256, 128, 128), (1000, 37, 130), (4096, 512, 384),
                                   (65536, 512, 1024), (33, 1, 1)])
def test_tf32x3_vs_fp64(cuda, m, d, N):
    dT, dE = run(cuda, m, d, N)
    assert dT < 1e-4, dT          # north_star fp32-mode tolerance
    # 3xTF32 products are ~fp32-exact; what remains is fp32 accumulation in TMEM
    # over m terms (~2^-24 sqrt(m)); a single TF32 pass would sit near 1e-3
    assert dT < 2e-7 * np.sqrt(m) + 1e-6, dT
    assert dE < 1e-4, dE


def test_tf32x3_matches_oracle_projection(cuda):
    import torch
    m, d, N = 3000, 20, 40
    x = oracle.random_matrix(m, d + 5, 9)
    r = oracle.decompose(x, d)
    xn = oracle.random_matrix(m, N, 10)
    Y32 = torch.as_tensor(np.asfortranarray(r.Y.astype(np.float32)).T.copy(), device=cuda).t()
    X32 = torch.as_tensor(np.asfortranarray(xn.astype(np.float32)).T.copy(), device=cuda).t()
    ldpad = (m + 3) // 4 * 4
    Tn, err = rbd.project_batch_f32(Y32, X32)
    Tr, er = oracle.project_batch(r.Y.astype(np.float32).astype(np.float64),
                                  xn.astype(np.float32).astype(np.float64))
    scale = np.sqrt((xn.astype(np.float32).astype(np.float64) ** 2).sum(0))
    assert (np.abs(Tn.cpu().numpy() - Tr) / scale).max() < 1e-4
    assert ldpad % 4 == 0


def _inputs(cuda, m, d, N, seed=3):
    import torch
    g = torch.Generator(device=cuda)
    g.manual_seed(seed)
    Y = torch.linalg.qr(torch.randn(m, d, dtype=torch.float64, device=cuda, generator=g))[0]
    Xn = torch.randn(m, N, dtype=torch.float64, device=cuda, generator=g)
    return Y.to(torch.float32).t().contiguous().t(), Xn.to(torch.float32).t().contiguous().t()


@pytest.mark.parametrize("m,d,N,sk", [(4096, 512, 384, "1"), (4100, 300, 700, "1"), (8192, 256, 256, "2"),
                                      (65536, 512, 1024, "2"), (3000, 129, 130, "1"), (40, 200, 260, "1")])
def test_pair_kernel_bitwise_equals_single_cta(cuda, monkeypatch, m, d, N, sk):
    """The CTA-pair kernel (tcgen05 cta_group::2, 256 x 256 tiles) runs the
    same MMAs per k-block in the same order as the 128 x 128 kernel: at equal
    split-K, T_new and the Eq. 3 indicator agree bit for bit. Shapes with
    partial pair tiles in d (a peer CTA with no basis rows), in N and in m."""
    import torch
    Y32, X32 = _inputs(cuda, m, d, N)
    monkeypatch.setenv("RBD_K6_SPLITK", sk)
    monkeypatch.setenv("RBD_K6_PAIR", "0")
    T1, e1 = rbd.project_batch_f32(Y32, X32)
    monkeypatch.setenv("RBD_K6_PAIR", "1")
    T2, e2 = rbd.project_batch_f32(Y32, X32)
    torch.cuda.synchronize()
    assert torch.equal(T1, T2)
    assert torch.equal(e1, e2)


@pytest.mark.parametrize("m,d,N", [(4096, 512, 384), (65536, 512, 2048), (1000, 260, 300)])
def test_pair_kernel_default_vs_fp64(cuda, m, d, N):
    """Library defaults (pair kernel, its own split-K choice) against fp64."""
    dT, dE = run(cuda, m, d, N, seed=5)
    assert dT < 2e-7 * np.sqrt(m) + 1e-6, dT
    assert dE < 1e-4, dE
