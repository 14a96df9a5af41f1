"""Forced-selection mode (SURVEY §8(c) parity protocol, rbd_set_forced_selection):
after an admissible near-tie divergence the B200 loop is re-run on the oracle's
selection so Y, T and the residual history are compared over ALL steps.
Near-duplicate column pairs make every pick a near tie."""
import numpy as np
import pytest
import torch

import oracle
import paper_1503_05947_b200 as rbd
from parity import compare

pytestmark = pytest.mark.gpu


def near_duplicates(m, n0, seed, rel=1e-15):
    a = oracle.random_matrix(m, n0, seed)
    return np.hstack([a, a + rel * oracle.random_matrix(m, n0, seed + 1)])


def test_forced_selection_full_length_parity(cuda):
    x = near_duplicates(300, 40, 3)
    r = oracle.decompose(x, 40)
    g = rbd.decompose(x, d_max=40, forced_selection=r.selected)
    assert g.selected == r.selected and g.d == r.d
    assert compare(g, r, x) == r.d
    # the protocol entry point: a free run, re-run on the oracle's picks if it diverges
    free = rbd.decompose(x, d_max=40)
    n = compare(free, r, x, rerun=lambda sel: rbd.decompose(x, d_max=40, forced_selection=sel))
    assert n == r.d


def test_forced_selection_arbitrary_sequence_matches_direct_projection(cuda):
    # any valid sequence: T = Y'X, Y orthonormal, history = max running residual
    x = oracle.random_matrix(512, 64, 5)
    seq = [7, 3, 60, 0, 33, 12, 41, 9]
    g = rbd.decompose(x, d_max=8, forced_selection=seq)
    assert g.selected == seq
    Y, T = np.asarray(g.Y), np.asarray(g.T)
    assert np.abs(Y.T @ Y - np.eye(8)).max() < 1e-13
    scale = np.linalg.norm(x, axis=0).max()
    assert np.abs(T - Y.T @ x).max() < 1e-12 * scale
    r = np.einsum("ij,ij->j", x, x) - np.cumsum(T * T, axis=0)
    hist = np.sqrt(np.maximum(r.max(axis=1), 0.0))
    np.testing.assert_allclose(g.residual_history, hist, rtol=1e-9, atol=1e-12 * scale)
    # the setting is cleared after the call: a later free run is greedy again
    assert rbd.decompose(x, d_max=8).selected == oracle.decompose(x, 8).selected


def test_forced_selection_weighted_persistent(monkeypatch, cuda):
    monkeypatch.setenv("RBD_DIAG_PATH", "persistent")
    x = near_duplicates(256, 30, 11)
    dg = oracle.random_positive(256, 12)
    r = oracle.decompose(x, 30, diag=dg)
    g = rbd.decompose(x, d_max=30, diag=dg, forced_selection=r.selected)
    assert g.selected == r.selected
    assert compare(g, r, x, diag=dg) == r.d


def test_forced_selection_device_entry(cuda):
    x = near_duplicates(128, 24, 21)
    r = oracle.decompose(x, 20)
    xd = torch.from_numpy(np.asfortranarray(x)).cuda()
    g = rbd.decompose(xd, d_max=20, forced_selection=r.selected)
    assert g.selected == r.selected
    assert compare(g, r, x) == r.d


def test_forced_selection_errors(monkeypatch, cuda):
    x = oracle.random_matrix(64, 16, 31)
    with pytest.raises(rbd.IndexOutOfRange):
        rbd.decompose(x, d_max=4, forced_selection=[0, 16])
    monkeypatch.setenv("RBD_PATH", "graph")
    ctx = rbd.Context(0)
    with pytest.raises(rbd.InvalidArgument):
        rbd.decompose(x, d_max=4, forced_selection=[0, 1], ctx=ctx)
    monkeypatch.delenv("RBD_PATH")
    # cleared after the call: the default context runs greedily again
    g = rbd.decompose(x, d_max=4)
    assert g.selected == oracle.decompose(x, 4).selected
