"""RBD1 container from and to HBM: a device-resident model larger
than one pinned staging buffer (32 MiB) streams through the double-buffered
D2H/H2D pipeline; bytes equal the oracle's restatement of io.cpp:533-570."""
import numpy as np
import pytest
import torch

import oracle
import paper_1503_05947_b200 as rbd

pytestmark = pytest.mark.gpu


def test_device_model_round_trip(cuda, tmp_path):
    g = torch.Generator(device="cuda").manual_seed(5)
    m, n, d = 32256, 700, 160                          # Y = 41 MB: two staging chunks
    X = (torch.randn(m, 24, generator=g, device="cuda", dtype=torch.float64)
         @ torch.randn(24, n, generator=g, device="cuda", dtype=torch.float64)
         + 1e-3 * torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64))
    X = X.t().contiguous().t()
    model = rbd.decompose(X, d_max=d)
    p = tmp_path / "dev.rbd"
    model.save(p, eps_r=0.25)
    Yh = model.Y.cpu().numpy()
    Th = model.T.cpu().numpy()
    assert p.read_bytes() == oracle.model_bytes(Yh, Th, 0.25, model.residual_history, 0)
    back, eps = rbd.load(p, device="cuda")
    assert eps == 0.25 and back.d == model.d
    assert back.Y.is_cuda and torch.equal(back.Y, model.Y) and torch.equal(back.T, model.T)
    host, _ = rbd.load(p)
    assert np.array_equal(host.Y, Yh) and np.array_equal(host.T, Th)


def test_device_diag_model_round_trip(cuda, tmp_path):
    x = oracle.random_matrix(3000, 120, 9)
    dg = oracle.random_positive(3000, 10)
    xd = torch.from_numpy(np.asfortranarray(x)).cuda()
    model = rbd.decompose(xd, d_max=40, diag=torch.from_numpy(dg).cuda())
    p = tmp_path / "diag.rbd"
    model.save(p, eps_r=0.0)
    assert p.read_bytes() == oracle.model_bytes(model.Y.cpu().numpy(), model.T.cpu().numpy(),
                                                0.0, model.residual_history, 1, dg)
    back, _ = rbd.load(p, device="cuda")
    assert back.weight_kind == 1 and np.array_equal(back.diag, dg)
    assert torch.equal(back.T, model.T)
