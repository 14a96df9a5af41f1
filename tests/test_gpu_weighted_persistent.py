"""Diagonal weight on the persistent loop (k_rbd_persistent<VEC, false, DIAG>,
SURVEY §8(f) row f1): the same oracle parity protocol as test_gpu_weighted.py
(workspace.cpp:24-29,61-99,114-122 restated in oracle/), with the path forced
by RBD_DIAG_PATH=persistent; agreement with the host-driven weighted steps;
the default gate picks the persistent loop at C1-like shapes."""
import numpy as np
import pytest
import torch

import oracle
import paper_1503_05947_b200 as rbd
from parity import compare, orthonormality_defect

pytestmark = pytest.mark.gpu


@pytest.fixture
def persistent(monkeypatch, cuda):
    monkeypatch.setenv("RBD_DIAG_PATH", "persistent")


def both(x, d_max, dg, eps=0.0, **kw):
    g = rbd.decompose(x, d_max=d_max, eps_r=eps, diag=dg, **kw)
    r = oracle.decompose(x, d_max, eps, diag=dg, **kw)
    return g, r


@pytest.mark.parametrize("m,n,d,seed", [(300, 80, 30, 1), (1024, 512, 64, 2), (33, 17, 12, 3),
                                        (4097, 9, 9, 4), (8193, 40, 25, 5), (5, 3, 3, 6),
                                        (64, 2, 2, 7), (4095, 333, 70, 8)])
def test_parity_random(persistent, m, n, d, seed):
    x = oracle.random_matrix(m, n, 100 + seed)
    dg = oracle.random_positive(m, 200 + seed)
    g, r = both(x, d, dg)
    rerun = lambda sel: rbd.decompose(x, d_max=d, diag=dg, forced_selection=sel)  # noqa: E731
    assert compare(g, r, x, diag=dg, rerun=rerun) == r.d
    assert g.result.launches < 8   # one persistent launch (+ init), not 12 per step


def test_parity_low_rank_with_noise(persistent):
    # noise well above the cancellation level of colsq_A - 2 cross + quad (~eps |x|^2):
    # at 1e-9 the post-rank argmax is decided by rounding on either path
    x = oracle.random_low_rank(200, 60, 8, 31) + 1e-6 * oracle.random_matrix(200, 60, 32)
    dg = oracle.random_positive(200, 33)
    g, r = both(x, 30, dg, eps=1e-12)
    compare(g, r, x, diag=dg)
    assert orthonormality_defect(g.Y) < 1e-12


@pytest.mark.parametrize("kw", [dict(reorthogonalize=True), dict(start_column=7),
                                dict(start_seed=12345), dict(breakdown_tol=1e-3)])
def test_parity_config_variants(persistent, kw):
    x = oracle.random_matrix(150, 40, 41)
    dg = oracle.random_positive(150, 42)
    g, r = both(x, 20, dg, **kw)
    assert compare(g, r, x, diag=dg) == r.d


def test_matches_host_driven_steps(monkeypatch, cuda):
    x = oracle.random_matrix(2048, 300, 71)
    dg = oracle.random_positive(2048, 72)
    monkeypatch.setenv("RBD_DIAG_PATH", "steps")
    s = rbd.decompose(x, d_max=60, diag=dg)
    monkeypatch.setenv("RBD_DIAG_PATH", "persistent")
    p = rbd.decompose(x, d_max=60, diag=dg)
    assert s.result.launches > 10 * p.result.launches
    assert p.selected == s.selected
    scale = np.linalg.norm(x, axis=0).max()
    np.testing.assert_allclose(p.T, s.T, rtol=0, atol=1e-11 * scale)
    np.testing.assert_allclose(p.residual_history, s.residual_history, rtol=1e-9, atol=1e-12 * scale)


def test_deterministic_and_device_entry(persistent):
    x = oracle.random_matrix(1500, 120, 81)
    dg = oracle.random_positive(1500, 82)
    a = rbd.decompose(x, d_max=40, diag=dg)
    xd = torch.from_numpy(np.asfortranarray(x)).cuda()
    b = rbd.decompose(xd, d_max=40, diag=torch.from_numpy(dg).cuda())
    assert a.selected == b.selected
    np.testing.assert_array_equal(a.Y, b.Y.cpu().numpy())
    np.testing.assert_array_equal(a.T, b.T.cpu().numpy())
    assert a.residual_history == b.residual_history


def test_default_gate_picks_persistent_at_scale(cuda):
    # d^2 <= m n / 256: one launch; Y orthonormal, T = Y'X, history = direct A-norm errors
    m, n, d = 8192, 1024, 96
    gen = torch.Generator(device="cuda").manual_seed(91)
    X = torch.randn(n, m, generator=gen, device="cuda", dtype=torch.float64).t()
    dg = torch.rand(m, generator=gen, device="cuda", dtype=torch.float64) * 2.0 + 0.5
    g = rbd.decompose(X, d_max=d, diag=dg)
    assert g.d == d and g.result.launches < 8
    Y, T = g.Y, g.T
    eye = torch.eye(d, device="cuda", dtype=torch.float64)
    assert float((Y.t() @ Y - eye).abs().max()) < 1e-12
    scale = float(X.norm(dim=0).max())
    assert float((T - Y.t() @ X).abs().max()) < 1e-11 * scale
    R = X - Y @ T
    e2 = ((R * R) * dg[:, None]).sum(0)
    # history[k] = sqrt(max_j e2_j) after k+1 vectors: check the last one
    assert abs(float(e2.max().sqrt()) - g.residual_history[-1]) < 1e-9 * scale
