"""K5 (out-of-sample compression T_new = Y'X_new, decompose.cpp:113-117, and
the Eq. 3 error indicator, workspace.cpp:88-97) under its three staging modes:
RBD_K5_TMA=0 per-thread cp.async, 1 TMA with 3 stages / 4 CTAs per SM, 2 TMA
with 4 stages / 3 CTAs per SM (the default). Oracle parity on ragged shapes
(partial 64-row / 64-column tiles, m not a multiple of 16, split-K boundaries,
padded leading dimensions), and bit-identity of T_new between staging modes
that use the same split-K factor (same K order, k = 4t + q per stage)."""
import numpy as np
import pytest

import oracle
import paper_1503_05947_b200 as rbd

pytestmark = pytest.mark.gpu


def dev(a, cuda, pad=0):
    import torch
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    buf = torch.zeros((a.shape[1], a.shape[0] + pad), dtype=torch.float64, device=cuda)
    buf[:, :a.shape[0]] = torch.as_tensor(a.T.copy(), device=cuda)
    return buf.t()[:a.shape[0]]


def basis(m, d, seed):
    q, _ = np.linalg.qr(oracle.random_matrix(m, d, seed))
    return np.asfortranarray(q)


SHAPES = [(1000, 37, 50), (65, 64, 130), (4097, 5, 3), (33, 1, 1), (16, 64, 64), (17, 65, 65),
          (3000, 130, 257), (8191, 200, 70)]


@pytest.mark.parametrize("mode", ["0", "1", "2"])
@pytest.mark.parametrize("m,d,N", SHAPES)
def test_k5_staging_vs_oracle(cuda, monkeypatch, mode, m, d, N):
    monkeypatch.setenv("RBD_K5_TMA", mode)
    y = basis(m, d, 40 + m)
    xn = oracle.random_matrix(m, N, 41 + N)
    Tn, err = rbd.project_batch(dev(y, cuda), dev(xn, cuda))
    Tr, er = oracle.project_batch(y, xn)
    scale = np.sqrt((xn * xn).sum(0))
    assert (np.abs(Tn.cpu().numpy() - Tr) / scale).max() < 1e-12
    assert (np.abs(err.cpu().numpy() - er) / (scale * scale)).max() < 1e-12


@pytest.mark.parametrize("pad", [2, 6])
def test_k5_tma_padded_leading_dimension(cuda, monkeypatch, pad):
    """ld > m (even, so the TMA strides stay 16-byte multiples)."""
    monkeypatch.setenv("RBD_K5_TMA", "2")
    m, d, N = 2050, 70, 90
    y = basis(m, d, 7)
    xn = oracle.random_matrix(m, N, 8)
    Tn, err = rbd.project_batch(dev(y, cuda, pad), dev(xn, cuda, pad + 2))
    Tr, er = oracle.project_batch(y, xn)
    scale = np.sqrt((xn * xn).sum(0))
    assert (np.abs(Tn.cpu().numpy() - Tr) / scale).max() < 1e-12
    assert (np.abs(err.cpu().numpy() - er) / (scale * scale)).max() < 1e-12


def test_k5_odd_leading_dimension_falls_back(cuda, monkeypatch):
    """An odd ld cannot be described to the TMA unit: the scalar K5 runs."""
    monkeypatch.setenv("RBD_K5_TMA", "2")
    m, d, N = 301, 9, 11
    y = basis(m, d, 3)
    xn = oracle.random_matrix(m, N, 4)
    Tn, _ = rbd.project_batch(dev(y, cuda), dev(xn, cuda))   # ld = m = 301
    Tr, _ = oracle.project_batch(y, xn)
    assert np.abs(Tn.cpu().numpy() - Tr).max() < 1e-12 * np.sqrt((xn * xn).sum(0)).max()


def test_k5_tma_bitwise_equals_cp_async(cuda, monkeypatch):
    """Modes 0 and 1 share the split-K factor (4 CTAs per SM) and the K order:
    identical T_new bits, multi-split, partial tiles."""
    import torch
    m, d, N = 20000, 130, 700
    g = torch.Generator(device="cuda").manual_seed(5)
    Y = torch.linalg.qr(torch.randn(m, d, dtype=torch.float64, device=cuda, generator=g))[0]
    X = torch.randn(N, m, dtype=torch.float64, device=cuda, generator=g).t()
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("RBD_K5_TMA", mode)
        out[mode] = rbd.project_batch(Y, X)
    assert torch.equal(out["0"][0], out["1"][0])
    ref = Y.t() @ X
    assert float((out["1"][0] - ref).abs().max()) < 1e-12 * float(X.norm(dim=0).max())
