"""Pins the oracle's diagonal-weight path to the reference's
own tests for that weight:

* proj/tests/test_workspace.cpp:39-60   col_sq = diag(X'AX) for a diagonal A (1e-12)
* proj/tests/test_workspace.cpp:62-66   init rejects a weight of the wrong dimension
* proj/tests/test_decompose.cpp:88-111  certification: a stop at eps_R bounds every
                                        column's A-norm residual (diagonal kind)
* proj/tests/test_decompose.cpp:113-126 the history equals directly computed A-norm
                                        errors (1e-7 relative)
* proj/tests/test_decompose.cpp:182-198 IncompatibleWeight for a 9-entry diagonal on m=10
* proj/tests/test_decompose.cpp:208-229 a diagonal weight steers the greedy selection
* proj/tests/acceptance.cpp:185-231     error_sq (offline-online identity) vs the direct
                                        residual, |fast - direct| <= 1e-9 max(1, col_sq),
                                        on seeded instances of the same shape family
* proj/src/weight.cpp:11-17             non-positive / non-finite / empty diagonals
"""
import numpy as np
import pytest

import oracle


def a_norm_sq(r, diag):  # weight.cpp:108-110,123-130 for a diagonal weight
    return max(float(np.dot(diag * r, r)), 0.0)


def test_random_positive_draws_are_reproducible():
    a = oracle.random_positive(12, 1041)
    assert np.array_equal(a, oracle.random_positive(12, 1041))
    assert a.min() >= 0.5 and a.max() < 3.0


def test_workspace_col_sq_equals_weighted_gram_diagonal():     # test_workspace.cpp:39-60
    m, n = 11, 6
    x = oracle.random_matrix(m, n, 11)
    dg = oracle.random_positive(m, 12)
    ws = oracle.Workspace(x, diag=dg)
    direct = np.einsum("ij,i,ij->j", x, dg, x)
    np.testing.assert_allclose(ws.col_sq(), direct, rtol=1e-12)
    np.testing.assert_array_equal(ws.residual(), ws.col_sq())


def test_workspace_rejects_wrong_dimension():                   # test_workspace.cpp:62-66
    x = oracle.random_matrix(5, 3, 14)
    with pytest.raises(oracle.OracleError) as e:
        oracle.Workspace(x, diag=np.ones(4))
    assert e.value.code == 2


def test_decompose_rejects_wrong_dimension():                   # test_decompose.cpp:196-198
    x = oracle.random_matrix(10, 6, 310)
    with pytest.raises(oracle.OracleError) as e:
        oracle.decompose(x, 2, diag=np.ones(9))
    assert e.value.code == 2


@pytest.mark.parametrize("bad", [np.array([1.0, 0.0, 2.0]), np.array([1.0, -1.0, 2.0]),
                                 np.array([1.0, np.inf, 2.0]), np.array([1.0, np.nan, 2.0]),
                                 np.array([])])
def test_diagonal_weight_validation(bad):                       # weight.cpp:11-17
    x = oracle.random_matrix(3, 3, 1)
    with pytest.raises(oracle.OracleError) as e:
        oracle.decompose(x, 2, diag=bad)
    assert e.value.code == 1


def test_certification_diagonal():                              # test_decompose.cpp:88-111
    eps = 1e-5
    base = oracle.random_low_rank(40, 25, 6, 250)
    x = base / np.linalg.norm(base) + 1e-7 * oracle.random_matrix(40, 25, 251)
    dg = oracle.random_positive(40, 252)
    model = oracle.decompose(x, 25, eps, diag=dg)
    assert model.residual_history[-1] <= eps
    assert model.d < 25
    for j in range(25):
        r = x[:, j] - model.Y @ model.T[:, j]
        assert np.sqrt(a_norm_sq(r, dg)) <= eps + 1e-10


def test_history_matches_direct_errors():                       # test_decompose.cpp:113-126
    x = oracle.random_matrix(20, 15, 260)
    dg = oracle.random_positive(20, 261)
    model = oracle.decompose(x, 8, diag=dg)
    worst = max(np.sqrt(a_norm_sq(x[:, j] - model.Y @ model.T[:, j], dg)) for j in range(15))
    assert model.residual_history[-1] == pytest.approx(worst, rel=1e-7)
    # every step's E_cur is the A-norm max over the columns after that step
    for d in range(1, model.d + 1):
        Yd, Td = model.Y[:, :d], model.T[:d]
        e = max(np.sqrt(a_norm_sq(x[:, j] - Yd @ Td[:, j], dg)) for j in range(15))
        assert model.residual_history[d - 1] == pytest.approx(e, rel=1e-7)


def test_diagonal_weight_steers_selection():                    # test_decompose.cpp:208-229
    x = np.zeros((4, 3))
    x[0, 0] = 1.0
    x[1, 1] = 2.0
    x[2, 2] = 0.5
    w = np.array([100.0, 1.0, 1.0, 1.0])
    plain = oracle.decompose(x, 2, start_column=2)
    assert plain.selected[1] == 1
    steered = oracle.decompose(x, 2, start_column=2, diag=w)
    assert steered.selected[1] == 0


def test_y_and_t_are_euclidean():
    # the weight enters only the error bookkeeping (workspace.cpp:61-99): Y stays
    # Euclidean-orthonormal and T = Y'X (decompose.cpp:88-93)
    x = oracle.random_matrix(30, 20, 7)
    dg = oracle.random_positive(30, 8)
    model = oracle.decompose(x, 10, diag=dg)
    assert np.abs(model.Y.T @ model.Y - np.eye(model.d)).max() < 1e-12
    assert np.abs(model.T - model.Y.T @ x).max() < 1e-12


@pytest.mark.parametrize("instance", range(24))
def test_offline_online_identity_diagonal(instance):           # acceptance.cpp:185-231 (diag)
    rng = np.random.default_rng(1000 + instance)
    m = int(rng.integers(5, 41))
    n = int(rng.integers(4, 31))
    d = 1 + int(rng.integers(0, min(10, m, n)))
    dg = rng.uniform(0.25, 4.0, m)
    x = oracle.random_matrix(m, n, 5000 + instance)
    model = oracle.decompose(x, d, diag=dg)
    ws = oracle.Workspace(x, diag=dg)
    for k in range(model.d):
        ws.extend(model.Y[:, k])
    np.testing.assert_allclose(ws.yay(), model.Y.T @ (dg[:, None] * model.Y), atol=1e-12)
    for j in range(n):
        c = model.T[:, j].copy()
        if instance % 2 == 1:
            c += rng.uniform(-0.5, 0.5, c.shape)
        fast = ws.error_sq(j, c)
        direct = a_norm_sq(x[:, j] - model.Y @ c, dg)
        assert abs(fast - direct) <= 1e-9 * max(1.0, ws.col_sq()[j])
    # residual_scan (general path) reproduces the decompose's last E_cur
    e, arg = ws.scan_T(model.T)
    assert e == model.residual_history[-1]
