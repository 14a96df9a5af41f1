"""GPU parity tests of the fp32 storage mode of rbd::decompose
(rbd_decompose_device_f32 / rbd_decompose_host_f32; BASELINE north_star's
optional fp32 mode).

X is held in fp32 and every product and sum is fp64 on the exact value of
each element, so the B200 result must equal the fp64 oracle run on the
fp32-valued matrix to the fp64 parity tolerances (1e-10, tests/parity.py).
Against the fp64 oracle on the unrounded matrix the bar is the north star's
fp32 tolerance, 1e-4 with the same scalings; there the admissible near-tie
gap is the fp32 input perturbation (tau = 1e-6 of max col_sq), not roundoff."""
import os

import numpy as np
import pytest

import oracle
import paper_1503_05947_b200 as rbd
from paper_1503_05947_b200 import configs
from parity import compare, orthonormality_defect

pytestmark = pytest.mark.gpu


def f32(x):
    return np.asfortranarray(np.asarray(x, dtype=np.float32))


def run_both(X32, d_max, eps=0.0, **kw):
    g = rbd.decompose(X32, d_max=d_max, eps_r=eps, **kw)
    r = oracle.decompose(X32.astype(np.float64), d_max, eps, **kw)
    return g, r


def test_c0_f32_equals_fp64_oracle_on_rounded_input(cuda):
    X32 = f32(configs.c0_matrix())
    g, r = run_both(X32, 64, 1e-6)
    assert g.d == r.d == 64
    rerun = lambda sel: rbd.decompose(X32, d_max=64, eps_r=1e-6, forced_selection=sel)  # noqa: E731
    assert compare(g, r, X32, rerun=rerun) == 64


@pytest.mark.parametrize("m,n,d", [(17, 12, 6), (1, 5, 1), (3, 1, 1), (4097, 9, 9), (8193, 7, 7),
                                   (4095, 33, 20), (12289, 130, 40), (5, 4, 4), (4098, 11, 8),
                                   (8192, 40, 16)])
def test_f32_shapes_parity(cuda, m, n, d):
    """m % 4 != 0 (scalar groups at the tail), partial last chunk, several
    chunks, n below the tile width, single row / column."""
    X32 = f32(oracle.random_matrix(m, n, 2000 + m + n))
    g, r = run_both(X32, d)
    rerun = lambda sel: rbd.decompose(X32, d_max=d, forced_selection=sel)  # noqa: E731
    assert compare(g, r, X32, rerun=rerun) == r.d


def test_f32_device_host_and_unaligned_ld_agree_bitwise(cuda):
    """Host entry, device entry with ld = m (float4 loads) and a device entry
    with an odd leading dimension (predicated scalar loads) give identical bits."""
    import torch
    m, n = 8200, 70
    X32 = f32(oracle.random_matrix(m, n, 91))
    a = rbd.decompose(X32, d_max=30)
    Xd = torch.as_tensor(np.ascontiguousarray(X32.T), device=cuda).t()
    b = rbd.decompose(Xd, d_max=30)
    buf = torch.zeros((n, m + 3), dtype=torch.float32, device=cuda)
    buf[:, :m] = torch.as_tensor(np.ascontiguousarray(X32.T), device=cuda)
    Xu = buf.t()[:m]
    assert Xu.stride() == (1, m + 3)
    c = rbd.decompose(Xu, d_max=30)
    for o in (b, c):
        assert a.selected == o.selected
        assert np.array_equal(a.Y, o.Y.cpu().numpy())
        assert np.array_equal(a.T, o.T.cpu().numpy())
        assert a.residual_history == o.residual_history


def test_f32_mode_matches_fp64_input_to_fp32_tolerance(cuda):
    """Against the fp64 oracle on the UNROUNDED matrix: the north star's 1e-4."""
    X = configs.c0_matrix(m=2048, n=256, rank=32, seed=3)
    X32 = f32(X)
    g = rbd.decompose(X32, d_max=32, eps_r=1e-6)
    r = oracle.decompose(X, 32, 1e-6)
    rerun = lambda sel: rbd.decompose(X32, d_max=32, eps_r=1e-6, forced_selection=sel)  # noqa: E731
    assert compare(g, r, X, tol=1e-4, tau=1e-6, rerun=rerun) == r.d


def test_f32_storage_flag_on_fp64_input(cuda):
    """storage='f32' on fp64 input rounds X to fp32 first: same bits as fp32 input."""
    X = oracle.random_matrix(600, 40, 5)
    a = rbd.decompose(X, d_max=12, storage="f32")
    b = rbd.decompose(f32(X), d_max=12)
    assert a.selected == b.selected and np.array_equal(a.Y, b.Y) and np.array_equal(a.T, b.T)
    c = rbd.decompose(f32(X), d_max=12, storage="f64")   # fp64 path on the same values
    assert c.selected == a.selected
    assert np.abs(c.Y - a.Y).max() < 1e-12


def test_f32_gating(cuda):
    x = f32(oracle.random_matrix(10, 6, 310))
    with pytest.raises(rbd.DegenerateInput):
        rbd.decompose(np.zeros((4, 3), dtype=np.float32), d_max=2)
    with pytest.raises(rbd.InvalidArgument):
        rbd.decompose(x, d_max=0)
    with pytest.raises(rbd.InvalidArgument):
        rbd.decompose(x, d_max=7)
    xn = x.copy()
    xn[3, 2] = np.nan
    with pytest.raises(rbd.InvalidArgument):
        rbd.decompose(xn, d_max=2)
    xi = x.copy()
    xi[0, 0] = np.inf
    with pytest.raises(rbd.InvalidArgument):
        rbd.decompose(xi, d_max=2)
    with pytest.raises(rbd.InvalidArgument):     # the fp32 mode is identity-only
        rbd.decompose(x, d_max=2, diag=np.ones(10), storage="f32")
    z = x.copy()
    z[:, 0] = 0.0
    with pytest.raises(rbd.DegenerateInput):
        rbd.decompose(z, d_max=2, breakdown_tol=1e-12)


def test_c1_f32_prefix_parity_and_full_properties(cuda):
    """C1 at full size in fp32 storage: the first 24 steps against the fp64
    oracle on the fp32-valued matrix, then size-independent properties of the
    whole 400-step run."""
    w = configs.C1
    Xd = configs.c1_matrix(n=w.n, seed=w.seed, device=cuda).float()
    X32 = np.asfortranarray(Xd.cpu().numpy())
    X = X32.astype(np.float64)
    eps = configs.eps_for(w, float(np.sqrt((X * X).sum(0)).max()))
    g = rbd.decompose(Xd, d_max=w.d_max, eps_r=eps)
    r = oracle.decompose(X, w.d_max, eps, nthreads=os.cpu_count() or 1, max_steps=24)

    class Prefix:
        pass
    gp = Prefix()
    gp.Y, gp.T, gp.d = g.Y[:, :r.d], g.T[:r.d], r.d
    gp.selected, gp.residual_history = g.selected[:r.d], g.residual_history[:r.d]
    compare(gp, r, X)
    assert g.d == w.d_max
    Y, T = g.Y, g.T
    G = (Y.t() @ Y).cpu().numpy()
    assert np.abs(G - np.eye(g.d)).max() < 1e-10
    T_direct = (Y.t() @ Xd.double()).cpu().numpy()
    colnorm = np.sqrt((X * X).sum(0))
    assert (np.abs(T_direct - T.cpu().numpy()) / colnorm).max() < 1e-12
    h = np.asarray(g.residual_history)
    assert np.all(h[1:] <= h[:-1] + 1e-12 * colnorm.max())
    assert len(set(g.selected)) == g.d
    # the fp64 run on the same fp32 values: same selection, same basis
    g64 = rbd.decompose(Xd.double(), d_max=w.d_max, eps_r=eps)
    assert g64.selected == g.selected
    assert orthonormality_defect(g.Y.cpu().numpy()) < 1e-10
    assert float((g64.Y - g.Y).abs().max()) < 1e-9


@pytest.mark.parametrize("kw", [dict(start_seed=12345), dict(start_column=7), dict(reorthogonalize=True),
                                dict(breakdown_tol=1e-3)])
def test_f32_config_fields_match_oracle(cuda, kw):
    """RbdConfig fields (start spec, reorthogonalize, breakdown_tol) in the fp32
    storage mode: same bits as the fp64 oracle on the fp32 values (to 1e-10)."""
    X32 = f32(configs.c0_matrix(m=3000, n=200, rank=24, seed=9))
    g, r = run_both(X32, 24, 0.0, **kw)
    rerun = lambda sel: rbd.decompose(X32, d_max=24, forced_selection=sel, **kw)  # noqa: E731
    assert compare(g, r, X32, rerun=rerun) == r.d


def test_f32_certified_stop(cuda):
    """Stop at eps_R: every column's fp64 residual against the fp32 values is
    within eps (+ roundoff), as test_decompose.cpp:88-111 for fp64."""
    X32 = f32(configs.c0_matrix(m=2048, n=300, rank=20, seed=4))
    X = X32.astype(np.float64)
    eps = 5e-2   # just above the noise floor: stops after ~60 of 200 steps
    g = rbd.decompose(X32, d_max=200, eps_r=eps)
    assert g.d < 200 and g.residual_history[-1] <= eps
    R = X - g.Y @ g.T
    assert np.sqrt((R * R).sum(0)).max() <= eps + 1e-10 * np.sqrt((X * X).sum(0)).max()


def test_f32_host_entry_pinned_outputs_equal_device_entry(cuda):
    """Page-locked Y/T stream out of the fp32 loop (host entry) with the same
    bits as the device entry."""
    import torch
    m, n, d = 20000, 600, 120
    X32 = f32(oracle.random_matrix(m, n, 17))
    a = rbd.decompose(X32, d_max=d)    # pinned outputs (>= 1 Mi elements)
    b = rbd.decompose(torch.as_tensor(np.ascontiguousarray(X32.T), device=cuda).t(), d_max=d)
    assert a.selected == b.selected
    assert np.array_equal(a.Y, b.Y.cpu().numpy()) and np.array_equal(a.T, b.T.cpu().numpy())


@pytest.mark.slow
def test_c2_f32_prefix_parity(cuda):
    """C2 (1 048 576 x 4 096) in fp32 storage at full size: the first 8 greedy
    steps against the fp64 oracle on the fp32-valued matrix."""
    import torch
    w = configs.C2
    Xd = configs.low_rank_matrix_torch(w.m, w.n, 1024, configs.spectrum("C2", 1024), 1e-8,
                                       w.seed, device=cuda)
    Xf = Xd.float()
    del Xd
    torch.cuda.empty_cache()
    g = rbd.decompose(Xf, d_max=8)
    Xh = torch.empty((w.n, w.m), dtype=torch.float32, pin_memory=True)
    Xh.copy_(Xf.t())
    del Xf
    X = Xh.numpy().T.astype(np.float64, order="F")
    r = oracle.decompose(X, 8, nthreads=os.cpu_count() or 1)

    class P:
        pass
    gp = P()
    gp.Y, gp.T, gp.d = g.Y.cpu().numpy(), g.T.cpu().numpy(), g.d
    gp.selected, gp.residual_history = g.selected, g.residual_history
    assert compare(gp, r, X) == 8


def test_f32_input_outside_the_fp32_mode_is_widened(cuda):
    """float32 input with a diagonal weight (or d_max above the persistent
    loop's limit) runs the fp64 path on the exactly widened values, as the
    reference's binding converts any array to a double Matrix
    (bindings.cpp:69-78); it is not rejected."""
    x = f32(oracle.random_matrix(40, 12, 311))
    w = oracle.random_positive(40, 312)
    a = rbd.decompose(x, d_max=6, diag=w)
    b = rbd.decompose(x.astype(np.float64), d_max=6, diag=w)
    assert a.selected == b.selected
    np.testing.assert_array_equal(a.Y, b.Y)
    np.testing.assert_array_equal(a.T, b.T)
    clf = rbd.fit(x, list(range(12)), d_max=6, diag=w)
    assert clf.predict(x[:, 3].astype(np.float64)) == 3
