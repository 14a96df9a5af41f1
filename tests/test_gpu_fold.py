"""GPU parity of the FOLD instantiation of the persistent loop (p_k = Y'w1_k
formed inside P1 from each CTA's row blocks). The library picks
it when Y outgrows L2 (C2, C4); RBD_FOLD=1 forces it on the small shapes here
and RBD_FOLD_KMAX switches steps between the fold and the Y'w1 sweep within
one decomposition. Oracle protocol and tolerances as tests/test_gpu_decompose.py."""
import numpy as np
import pytest

import oracle
import paper_1503_05947_b200 as rbd
from paper_1503_05947_b200 import configs
from parity import compare, orthonormality_defect

pytestmark = pytest.mark.gpu


@pytest.fixture
def fold_env(monkeypatch):
    monkeypatch.setenv("RBD_FOLD", "1")
    return monkeypatch


def test_c0_fold_parity(cuda, fold_env):
    X = configs.c0_matrix()
    g = rbd.decompose(X, d_max=64, eps_r=1e-6)
    r = oracle.decompose(X, 64, 1e-6)
    assert g.d == r.d == 64
    rerun = lambda sel: rbd.decompose(X, d_max=64, eps_r=1e-6, forced_selection=sel)  # noqa: E731
    assert compare(g, r, X, rerun=rerun) == 64


@pytest.mark.parametrize("m,n,d", [(4096, 40, 30), (8194, 33, 33), (12290, 130, 100), (700, 300, 160),
                                   (64, 200, 60), (2, 9, 2)])
def test_fold_shapes_parity(cuda, fold_env, m, n, d):
    """Even m (the fold needs 16-byte row pairs): a partial last P1 block,
    CTAs with no rows, k beyond one 128-column fold batch (reversed re-read
    order over several batches)."""
    X = oracle.random_matrix(m, n, 3000 + m + n)
    g = rbd.decompose(X, d_max=d)
    r = oracle.decompose(X, d)
    assert compare(g, r, X, rerun=lambda sel: rbd.decompose(X, d_max=d, forced_selection=sel)) == r.d


@pytest.mark.parametrize("kmax", ["0", "7", "33"])
def test_fold_kmax_switch_matches_oracle(cuda, fold_env, kmax):
    """Steps k <= RBD_FOLD_KMAX fold, later steps sweep Y: both kinds of
    step in one run, and the switch leaves the second pass intact."""
    fold_env.setenv("RBD_FOLD_KMAX", kmax)
    X = oracle.random_matrix(9000, 80, 55)
    g = rbd.decompose(X, d_max=60)
    r = oracle.decompose(X, 60)
    assert compare(g, r, X, rerun=lambda sel: rbd.decompose(X, d_max=60, forced_selection=sel)) == r.d
    assert orthonormality_defect(g.Y) < 1e-12


def test_fold_deterministic_and_close_to_unfolded(cuda, monkeypatch):
    """Bitwise run to run; against the Y'w1 sweep only the order of p_k's
    sums differs (same selections, Y/T at rounding level)."""
    X = oracle.random_matrix(20000, 96, 91)
    monkeypatch.setenv("RBD_FOLD", "1")
    a = rbd.decompose(X, d_max=80)
    b = rbd.decompose(X, d_max=80)
    assert a.selected == b.selected
    assert np.array_equal(a.Y, b.Y) and np.array_equal(a.T, b.T)
    monkeypatch.setenv("RBD_FOLD", "0")
    c = rbd.decompose(X, d_max=80)
    assert a.selected == c.selected
    assert np.abs(a.Y - c.Y).max() < 1e-12
    assert np.abs(a.T - c.T).max() < 1e-10 * np.sqrt((X * X).sum(0)).max()


def test_fold_rank_deficient_breakdown(cuda, fold_env):
    """Breakdown decided on the folded p_k: rank-5 matrix stops at d = 5 as
    the oracle does."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((3000, 5)) @ rng.standard_normal((5, 40))
    g = rbd.decompose(A, d_max=20)
    r = oracle.decompose(A, 20)
    assert g.d == r.d
    assert compare(g, r, A) == r.d


@pytest.mark.parametrize("m,n,d", [(8194, 40, 33), (12290, 130, 100)])
def test_fold_f32_storage_parity(cuda, fold_env, m, n, d):
    """The fp32 storage mode's FOLD instantiation (X in fp32, Y and the fold
    in fp64) against the fp64 oracle on the fp32-valued matrix, 1e-10."""
    X32 = np.asfortranarray(oracle.random_matrix(m, n, 4000 + m).astype(np.float32))
    g = rbd.decompose(X32, d_max=d)
    r = oracle.decompose(X32.astype(np.float64), d)
    assert compare(g, r, X32, rerun=lambda sel: rbd.decompose(X32, d_max=d, forced_selection=sel)) == r.d
