"""Diagonal-weight decompose on the B200 path through the C
ABI (rbd_decompose_diag_host / _device) against the oracle's restatement of
the reference's weighted bookkeeping (workspace.cpp:24-29,61-99,114-122) and
against the reference's own diagonal-weight tests (test_decompose.cpp:88-126,
182-229). Parity protocol: tests/parity.py with diag (A-norm near ties)."""
import numpy as np
import pytest
import torch

import oracle
import paper_1503_05947_b200 as rbd
from parity import compare, orthonormality_defect

pytestmark = pytest.mark.gpu


def a_norm_sq(r, dg):
    return max(float(np.dot(dg * r, r)), 0.0)


def both(x, d_max, dg, eps=0.0, **kw):
    g = rbd.decompose(x, d_max=d_max, eps_r=eps, diag=dg, **kw)
    r = oracle.decompose(x, d_max, eps, diag=dg, **kw)
    return g, r


@pytest.mark.parametrize("m,n,d,seed", [(300, 80, 30, 1), (1024, 512, 64, 2), (33, 17, 12, 3),
                                        (4097, 9, 9, 4), (8193, 40, 25, 5), (5, 3, 3, 6),
                                        (64, 2, 2, 7)])
def test_parity_random(cuda, m, n, d, seed):
    x = oracle.random_matrix(m, n, 100 + seed)
    dg = oracle.random_positive(m, 200 + seed)
    g, r = both(x, d, dg)
    assert compare(g, r, x, diag=dg) == r.d


def test_parity_low_rank_with_noise_floor(cuda):
    x = oracle.random_low_rank(200, 60, 8, 31) + 1e-9 * oracle.random_matrix(200, 60, 32)
    dg = oracle.random_positive(200, 33)
    g, r = both(x, 30, dg, eps=1e-12)
    compare(g, r, x, diag=dg)
    assert orthonormality_defect(g.Y) < 1e-12


@pytest.mark.parametrize("kw", [dict(reorthogonalize=True), dict(start_column=7),
                                dict(start_seed=12345), dict(breakdown_tol=1e-3)])
def test_parity_config_variants(cuda, kw):
    x = oracle.random_matrix(150, 40, 41)
    dg = oracle.random_positive(150, 42)
    g, r = both(x, 20, dg, **kw)
    assert compare(g, r, x, diag=dg) == r.d


def test_device_entry_matches_host_entry(cuda):
    x = oracle.random_matrix(512, 100, 51)
    dg = oracle.random_positive(512, 52)
    h = rbd.decompose(x, d_max=40, diag=dg)
    xd = torch.from_numpy(np.asfortranarray(x)).cuda()
    dv = rbd.decompose(xd, d_max=40, diag=torch.from_numpy(dg).cuda())
    assert h.selected == dv.selected
    np.testing.assert_array_equal(h.Y, dv.Y.cpu().numpy())
    np.testing.assert_array_equal(h.T, dv.T.cpu().numpy())
    assert h.residual_history == dv.residual_history


def test_deterministic(cuda):
    x = oracle.random_matrix(256, 90, 61)
    dg = oracle.random_positive(256, 62)
    a = rbd.decompose(x, d_max=30, diag=dg)
    b = rbd.decompose(x, d_max=30, diag=dg)
    assert a.selected == b.selected
    assert np.array_equal(a.Y, b.Y) and np.array_equal(a.T, b.T)


# ---------------- the reference's diagonal-weight tests ----------------

def test_certification_diagonal(cuda):                          # test_decompose.cpp:88-111
    eps = 1e-5
    base = oracle.random_low_rank(40, 25, 6, 250)
    x = base / np.linalg.norm(base) + 1e-7 * oracle.random_matrix(40, 25, 251)
    dg = oracle.random_positive(40, 252)
    model = rbd.decompose(x, d_max=25, eps_r=eps, diag=dg)
    assert model.residual_history[-1] <= eps
    assert model.d < 25
    for j in range(25):
        r = x[:, j] - model.Y @ model.T[:, j]
        assert np.sqrt(a_norm_sq(r, dg)) <= eps + 1e-10


def test_history_matches_direct_errors(cuda):                   # test_decompose.cpp:113-126
    x = oracle.random_matrix(20, 15, 260)
    dg = oracle.random_positive(20, 261)
    model = rbd.decompose(x, d_max=8, diag=dg)
    worst = max(np.sqrt(a_norm_sq(x[:, j] - model.Y @ model.T[:, j], dg)) for j in range(15))
    assert model.residual_history[-1] == pytest.approx(worst, rel=1e-7)


def test_diagonal_weight_steers_selection(cuda):                # test_decompose.cpp:208-229
    x = np.zeros((4, 3))
    x[0, 0] = 1.0
    x[1, 1] = 2.0
    x[2, 2] = 0.5
    w = np.array([100.0, 1.0, 1.0, 1.0])
    assert rbd.decompose(x, d_max=2, start_column=2).selected[1] == 1
    assert rbd.decompose(x, d_max=2, start_column=2, diag=w).selected[1] == 0


def test_gating(cuda):                                          # test_decompose.cpp:182-198
    x = oracle.random_matrix(10, 6, 310)
    with pytest.raises(rbd.IncompatibleWeight):
        rbd.decompose(x, d_max=2, diag=np.ones(9))
    with pytest.raises(rbd.InvalidArgument):                    # checked before the weight
        rbd.decompose(x, d_max=7, diag=np.ones(9))
    for bad in (np.array([]), np.r_[np.ones(9), 0.0], np.r_[np.ones(9), -1.0],
                np.r_[np.ones(9), np.nan], np.r_[np.ones(9), np.inf]):
        with pytest.raises(rbd.InvalidArgument):                # weight.cpp:11-17
            rbd.decompose(x, d_max=2, diag=bad)
    with pytest.raises(rbd.DegenerateInput):
        rbd.decompose(np.zeros((4, 3)), d_max=2, diag=np.ones(4))


def test_y_t_euclidean_and_history_direct_at_scale(cuda):
    # C1-shaped block (32 256 rows) with a smooth diagonal weight: Y orthonormal,
    # T = Y'X, and every step's E_cur equals the directly computed A-norm maximum
    m, n, d = 32256, 256, 40
    rng = np.random.default_rng(7)
    x = np.asfortranarray(rng.standard_normal((m, 12)) @ rng.standard_normal((12, n))
                          + 1e-3 * rng.standard_normal((m, n)))
    dg = 0.5 + np.linspace(0.0, 2.0, m)
    g = rbd.decompose(x, d_max=d, diag=dg)
    assert orthonormality_defect(g.Y) < 1e-12
    assert np.abs(g.T - g.Y.T @ x).max() <= 1e-12 * np.abs(x).max() * np.sqrt(m)
    # the A-norm bookkeeping col_sq_A - 2 cross + quad cancels at ~eps * col_sq_A
    # (as the reference's own does, test_decompose.cpp:89-90)
    colsq_a = np.einsum("ij,i,ij->j", x, dg, x)
    for k in (1, d // 2, g.d):
        R = x - g.Y[:, :k] @ g.T[:k]
        e2 = np.maximum(np.einsum("ij,i,ij->j", R, dg, R), 0.0).max()
        assert abs(g.residual_history[k - 1] ** 2 - e2) <= 1e-12 * colsq_a.max()


# ---------------- the diagonal ErrorWorkspace (rbd_ws_* with a weight) ----------------

def _cuda(x):
    return torch.from_numpy(np.asfortranarray(x)).cuda()


def test_workspace_col_sq_weighted(cuda):                        # test_workspace.cpp:39-60
    m, n = 11, 6
    x = oracle.random_matrix(m, n, 11)
    dg = oracle.random_positive(m, 12)
    ws = rbd.Workspace(_cuda(x), diag=dg)
    col_sq, resid, _ = ws.read()
    np.testing.assert_allclose(col_sq, np.einsum("ij,i,ij->j", x, dg, x), rtol=1e-12)
    np.testing.assert_array_equal(resid, col_sq)


def test_workspace_rejects_bad_weights(cuda):                    # test_workspace.cpp:62-66
    x = _cuda(oracle.random_matrix(5, 3, 14))
    with pytest.raises(rbd.IncompatibleWeight):
        rbd.Workspace(x, diag=np.ones(4))
    with pytest.raises(rbd.InvalidArgument):
        rbd.Workspace(x, diag=np.r_[np.ones(4), 0.0])


@pytest.mark.parametrize("instance", range(12))
def test_workspace_offline_online_identity(cuda, instance):      # acceptance.cpp:185-231 (diag)
    rng = np.random.default_rng(2000 + instance)
    m = int(rng.integers(5, 41))
    n = int(rng.integers(4, 31))
    d = 1 + int(rng.integers(0, min(10, m, n)))
    dg = rng.uniform(0.25, 4.0, m)
    x = oracle.random_matrix(m, n, 7000 + instance)
    model = oracle.decompose(x, d, diag=dg)
    ws = rbd.Workspace(_cuda(x), cap=d, diag=dg)
    ows = oracle.Workspace(x, diag=dg)
    for k in range(model.d):
        ws.extend(torch.from_numpy(model.Y[:, k].copy()).cuda())
        ows.extend(model.Y[:, k])
    np.testing.assert_allclose(ws.yay(), ows.yay(), rtol=0, atol=1e-12)
    _, _, yax = ws.read()
    for k in range(model.d):
        np.testing.assert_allclose(yax[k], ows.yax_row(k), rtol=0, atol=1e-12 * max(1, np.abs(x).max()))
    for j in range(n):
        c = model.T[:, j].copy()
        if instance % 2 == 1:
            c += rng.uniform(-0.5, 0.5, c.shape)
        fast = ws.error_sq(j, c)
        r = x[:, j] - model.Y @ c
        direct = max(float(np.dot(dg * r, r)), 0.0)
        assert abs(fast - direct) <= 1e-9 * max(1.0, ows.col_sq()[j])
    e, arg = ws.scan_T(model.T)
    e_ref, arg_ref = ows.scan_T(model.T)
    assert arg == arg_ref and e == pytest.approx(e_ref, rel=1e-9, abs=1e-12)


def test_workspace_scan_T_identity_matches_scan(cuda):
    x = oracle.random_matrix(60, 25, 9)
    model = oracle.decompose(x, 8)
    ws = rbd.Workspace(_cuda(x), cap=8)
    for k in range(model.d):
        ws.extend(torch.from_numpy(model.Y[:, k].copy()).cuda())
    e1, j1 = ws.scan()
    e2, j2 = ws.scan_T(model.T)
    assert j1 == j2 and e1 == pytest.approx(e2, rel=1e-9)
