"""GPU workspace (K1 init, K2 sweep, K3 scan) and out-of-sample projection (K5)
against the oracle and the reference's proj/tests/test_workspace.cpp (identity
weight cases), SPEC.md:201-204 and acceptance.cpp criterion 3."""
import numpy as np
import pytest

import oracle
import paper_1503_05947_b200 as rbd

pytestmark = pytest.mark.gpu


def dev(a, cuda):
    import torch
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if a.ndim == 1:
        return torch.as_tensor(a.copy(), device=cuda)
    return torch.as_tensor(a.T.copy(), device=cuda).t()


def orthonormal_basis(x, d):                       # test_workspace.cpp:17-27
    y = np.zeros((x.shape[0], d), order="F")
    have = 0
    for j in range(x.shape[1]):
        if have == d:
            break
        r = oracle.mgs_project(x[:, j], y[:, :have], 1e-10, True)
        if r is not None:
            y[:, have] = r[0]
            have += 1
    assert have == d
    return y


def test_init_col_sq(cuda):                        # :28-37
    x = np.array([[1.0, 0.0], [0.0, 2.0], [0.0, 0.0]])
    ws = rbd.Workspace(dev(x, cuda))
    col_sq, resid, _ = ws.read()
    assert col_sq[0] == 1.0 and col_sq[1] == 4.0
    assert np.array_equal(resid, col_sq)


def test_init_col_sq_matches_oracle(cuda):         # :39-62 (identity)
    for (m, n) in [(11, 6), (4097, 13), (10000, 5)]:
        x = oracle.random_matrix(m, n, 11 + m)
        ws = rbd.Workspace(dev(x, cuda))
        col_sq, _, _ = ws.read()
        ref = oracle.Workspace(x).col_sq()
        assert np.allclose(col_sq, ref, rtol=1e-12, atol=0)


def test_error_sq_vs_direct(cuda):                 # :68-95 (identity)
    m, n, d = 13, 7, 4
    x = oracle.random_matrix(m, n, 20)
    y = orthonormal_basis(x, d)
    t = y.T @ x
    ws = rbd.Workspace(dev(x, cuda), cap=d)
    for k in range(d):
        ws.extend(dev(y[:, k], cuda))
    assert ws.d == d
    col_sq, _, _ = ws.read()
    for j in range(n):
        exact = t[:, j]
        off = exact + 0.3 * oracle.random_matrix(d, 1, 23 + j)[:, 0]
        for c in (exact, off):
            r = x[:, j] - y @ c
            direct = r @ r
            assert abs(ws.error_sq(j, c) - direct) <= 1e-9 * max(1.0, col_sq[j])


def test_error_sq_gating(cuda):                    # :97-107
    x = oracle.random_matrix(6, 4, 30)
    y = orthonormal_basis(x, 2)
    ws = rbd.Workspace(dev(x, cuda), cap=4)
    ws.extend(dev(y[:, 0], cuda))
    ws.extend(dev(y[:, 1], cuda))
    with pytest.raises(rbd.IndexOutOfRange):
        ws.error_sq(-1, np.zeros(2))
    with pytest.raises(rbd.IndexOutOfRange):
        ws.error_sq(4, np.zeros(2))
    with pytest.raises(rbd.DimensionMismatch):
        ws.error_sq(0, np.zeros(3))


def test_scan_vs_exhaustive(cuda):                 # :124-153 (identity)
    m, n, d = 15, 9, 3
    x = oracle.random_matrix(m, n, 40)
    y = orthonormal_basis(x, d)
    t = y.T @ x
    ws = rbd.Workspace(dev(x, cuda), cap=d)
    for k in range(d):
        ws.extend(dev(y[:, k], cuda))
    e = [float((x[:, j] - y @ t[:, j]) @ (x[:, j] - y @ t[:, j])) for j in range(n)]
    best_j = int(np.argmax(e))
    e_cur, arg = ws.scan()
    assert arg == best_j
    assert abs(e_cur - np.sqrt(e[best_j])) <= 1e-7 * np.sqrt(e[best_j])


def test_scan_ties_smallest_index(cuda):           # :155-175
    x = oracle.random_matrix(8, 5, 50)
    x[:, 3] = x[:, 1]
    y = orthonormal_basis(x, 1)
    ws = rbd.Workspace(dev(x, cuda), cap=1)
    ws.extend(dev(y[:, 0], cuda))
    e_cur, arg = ws.scan()
    _, resid, _ = ws.read()
    assert resid[1] == resid[3]
    if resid[1] == resid.max():
        assert arg == 1


def test_scan_exact_ties_many(cuda):
    """Exact ties across CTAs / tiles: smallest index must win."""
    n = 5000
    x = np.zeros((4, n))
    x[0, :] = 1.0
    x[1, 1234] = 0.0
    ws = rbd.Workspace(dev(x, cuda))
    e_cur, arg = ws.scan()
    assert arg == 0 and e_cur == 1.0
    x[2, 4321] = 1.0
    x[2, 777] = 1.0
    ws = rbd.Workspace(dev(x, cuda))
    assert ws.scan()[1] == 777


def test_spec_scan_example(cuda):
    x = np.array([[1.0, 0.0], [0.0, 1.0]])
    ws = rbd.Workspace(dev(x, cuda), cap=1)
    ws.extend(dev(np.array([1.0, 0.0]), cuda))
    e_cur, arg = ws.scan()
    assert e_cur == 1.0 and arg == 1
    ws0 = rbd.Workspace(dev(np.zeros((3, 4)) + np.eye(3, 4), cuda), cap=3)
    for k in range(3):
        ws0.extend(dev(np.eye(3)[:, k], cuda))
    e0, a0 = ws0.scan()
    assert e0 == 0.0 and a0 == 0


def test_residuals_nonnegative_full_span(cuda):    # :200-212
    m, n = 20, 12
    x = oracle.random_matrix(m, n, 70)
    y = orthonormal_basis(x, n)
    ws = rbd.Workspace(dev(x, cuda), cap=n)
    for k in range(n):
        ws.extend(dev(y[:, k], cuda))
        assert ws.read()[1].min() >= 0.0
    assert ws.read()[1].max() < 1e-10


def test_workspace_matches_oracle_sequence(cuda):
    """Fixed Y sequence fed to both workspaces: T rows and residuals agree."""
    m, n, d = 9000, 37, 8
    x = oracle.random_matrix(m, n, 91)
    y = orthonormal_basis(x, d)
    g = rbd.Workspace(dev(x, cuda), cap=d)
    o = oracle.Workspace(x)
    for k in range(d):
        g.extend(dev(y[:, k], cuda))
        o.extend(y[:, k])
    col_sq, resid, yax = g.read()
    for k in range(d):
        assert np.abs(yax[k] - o.yax_row(k)).max() <= 1e-12 * np.sqrt(col_sq).max()
    assert np.abs(resid - o.residual()).max() <= 1e-10 * col_sq.max()
    assert g.scan()[1] == o.scan()[1]


# ---------------- out-of-sample compression ----------------

@pytest.mark.parametrize("m,d,N", [(1000, 37, 50), (65, 64, 130), (4097, 5, 3), (33, 1, 1)])
def test_project_batch_vs_oracle(cuda, m, d, N):
    x = oracle.random_matrix(m, max(d, 2) + 3, 5 + m)
    y = orthonormal_basis(x, d)
    xn = oracle.random_matrix(m, N, 6 + N)
    Tn, err = rbd.project_batch(dev(y, cuda), dev(xn, cuda))
    Tr, er = oracle.project_batch(y, xn)
    scale = np.sqrt((xn * xn).sum(0))
    assert (np.abs(Tn.cpu().numpy() - Tr) / scale).max() < 1e-12
    assert (np.abs(err.cpu().numpy() - er) / (scale * scale)).max() < 1e-12
    Th, eh = rbd.project_batch(y, xn)   # host entry
    assert np.array_equal(Th, Tn.cpu().numpy())


def test_project_error_indicator_identity(cuda):
    """err_j equals ||x - Y Y'x||^2 (Eq. 3) for in-span and off-span vectors."""
    m, d = 500, 20
    x = oracle.random_matrix(m, d, 9)
    y = orthonormal_basis(x, d)
    inside = y @ oracle.random_matrix(d, 4, 10)
    outside = oracle.random_matrix(m, 4, 11)
    xn = np.concatenate([inside, outside], axis=1)
    Tn, err = rbd.project_batch(dev(y, cuda), dev(xn, cuda))
    direct = ((xn - y @ (y.T @ xn)) ** 2).sum(0)
    colsq = (xn * xn).sum(0)
    assert np.abs(err.cpu().numpy() - direct).max() <= 1e-12 * colsq.max()
