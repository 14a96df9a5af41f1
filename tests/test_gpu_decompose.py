"""GPU parity tests: the B200 path (through the C ABI) against the CPU oracle
and against the reference's own hot-path tests, ported case by case from
proj/tests/test_decompose.cpp, acceptance.cpp criteria 1-4 and
proj/tests/python/test_smoke.py. Tolerances are the reference's own unless
stated; parity tolerance 1e-10 (fp64) per BASELINE.json north_star."""
import numpy as np
import pytest

import oracle
import paper_1503_05947_b200 as rbd
from paper_1503_05947_b200 import configs
from parity import compare, orthonormality_defect

pytestmark = pytest.mark.gpu


def basic(x, d_max, eps=0.0, **kw):
    return rbd.decompose(x, d_max=d_max, eps_r=eps, **kw)


def both(x, d_max, eps=0.0, **kw):
    g = rbd.decompose(x, d_max=d_max, eps_r=eps, **kw)
    r = oracle.decompose(x, d_max, eps, **kw)
    return g, r


# ---------------- oracle parity ----------------

def test_c0_parity_full(cuda):
    X = configs.c0_matrix()
    g, r = both(X, 64, 1e-6)
    assert g.d == r.d == 64
    rerun = lambda sel: rbd.decompose(X, d_max=64, eps_r=1e-6, forced_selection=sel)  # noqa: E731
    assert compare(g, r, X, rerun=rerun) == 64


@pytest.mark.parametrize("m,n,d", [(17, 12, 6), (1, 5, 1), (3, 1, 1), (4097, 9, 9), (8193, 7, 7),
                                   (4095, 33, 20), (12289, 130, 40), (5, 4, 4)])
def test_shapes_parity(cuda, m, n, d):
    """Edge shapes: odd m (scalar path), n < tile width, partial last chunk,
    multi-chunk rows, single row / single column."""
    X = oracle.random_matrix(m, n, 1000 + m + n)
    g, r = both(X, d)
    assert compare(g, r, X, rerun=lambda sel: rbd.decompose(X, d_max=d, forced_selection=sel)) == r.d


def test_padded_leading_dimension_device(cuda):
    import torch
    m, n = 1000, 50
    X = oracle.random_matrix(m, n, 77)
    buf = torch.zeros((n, m + 24), dtype=torch.float64, device=cuda)
    buf[:, :m] = torch.as_tensor(X.T, device=cuda)
    Xd = buf.t()[:m]                      # m x n, column stride m + 24
    assert Xd.stride() == (1, m + 24)
    g = rbd.decompose(Xd, d_max=20)
    r = oracle.decompose(X, 20)
    compare(g, r, X)


def test_device_and_host_entry_agree_bitwise(cuda):
    import torch
    X = configs.c0_matrix()
    a = rbd.decompose(X, d_max=32, eps_r=1e-6)
    Xd = torch.as_tensor(X.T.copy(), device=cuda).t()
    b = rbd.decompose(Xd, d_max=32, eps_r=1e-6)
    assert a.selected == b.selected
    assert np.array_equal(a.Y, b.Y.cpu().numpy())
    assert np.array_equal(a.T, b.T.cpu().numpy())
    assert a.residual_history == b.residual_history


def test_c1_parity_first_steps_and_full_properties(cuda):
    import torch
    w = configs.C1
    Xd = configs.c1_matrix(n=w.n, seed=w.seed, device=cuda)
    X = Xd.cpu().numpy()
    eps = configs.eps_for(w, float(np.sqrt((X * X).sum(0)).max()))
    g = rbd.decompose(Xd, d_max=w.d_max, eps_r=eps)
    import os
    r = oracle.decompose(X, w.d_max, eps, nthreads=os.cpu_count() or 1, max_steps=24)
    # parity over the oracle's bounded prefix
    class Prefix:
        pass
    gp = Prefix()
    gp.Y, gp.T, gp.d = g.Y[:, :r.d], g.T[:r.d], r.d
    gp.selected, gp.residual_history = g.selected[:r.d], g.residual_history[:r.d]
    compare(gp, r, X)
    # full-size, size-independent properties of the whole GPU run
    Y, T = g.Y, g.T
    assert g.d >= 24
    G = (Y.t() @ Y).cpu().numpy()
    assert np.abs(G - np.eye(g.d)).max() < 1e-10
    T_direct = (Y.t() @ Xd).cpu().numpy()
    colnorm = np.sqrt((X * X).sum(0))
    assert (np.abs(T_direct - T.cpu().numpy()) / colnorm).max() < 1e-12
    h = np.asarray(g.residual_history)
    assert np.all(h[1:] <= h[:-1] + 1e-12 * colnorm.max())
    if h[-1] <= eps:   # certified stop: every column within eps (+ roundoff)
        R = Xd - Y @ T
        assert float(R.norm(dim=0).max()) <= eps + 1e-10 * colnorm.max()
    assert len(set(g.selected)) == g.d


@pytest.mark.slow
def test_c1_full_parity_all_steps(cuda):
    """C1 at full size, all 400 greedy steps against the threaded oracle."""
    import os
    w = configs.C1
    Xd = configs.c1_matrix(n=w.n, seed=w.seed, device=cuda)
    X = np.asfortranarray(Xd.cpu().numpy())
    eps = configs.eps_for(w, float(np.sqrt((X * X).sum(0)).max()))
    g = rbd.decompose(Xd, d_max=w.d_max, eps_r=eps)
    r = oracle.decompose(X, w.d_max, eps, nthreads=os.cpu_count() or 1)
    assert compare(g, r, X) == r.d == g.d == w.d_max


def test_determinism_bitwise(cuda):
    X = configs.c0_matrix()
    a = basic(X, 64, 1e-6)
    b = basic(X, 64, 1e-6)
    assert a.selected == b.selected
    assert np.array_equal(a.Y, b.Y) and np.array_equal(a.T, b.T)
    assert a.residual_history == b.residual_history


# ---------------- ports of proj/tests/test_decompose.cpp ----------------

def test_rank1_outer_product(cuda):                       # :29-40
    u = oracle.random_matrix(30, 1, 100)[:, 0]
    v = oracle.random_matrix(20, 1, 101)[:, 0]
    x = np.outer(u, v)
    m = basic(x, 10, 1e-10)
    assert m.d == 1
    assert np.abs(x - m.Y @ m.T).max() < 1e-10
    assert abs(abs(m.Y[:, 0] @ (u / np.linalg.norm(u))) - 1.0) < 1e-12


@pytest.mark.parametrize("seed", [200, 201, 202])
def test_basis_orthonormal(cuda, seed):                   # :42-49
    x = oracle.random_matrix(25, 18, seed)
    m = basic(x, 12)
    assert m.d == 12
    assert orthonormality_defect(m.Y) < 1e-10


def test_rank_deficient_noise_floor(cuda):                # :51-57
    x = oracle.random_low_rank(40, 30, 5, 210)
    m = basic(x, 30)
    assert m.d == 5
    assert orthonormality_defect(m.Y) < 1e-10
    assert np.abs(x - m.Y @ m.T).max() < 1e-9


def test_history_monotone(cuda):                          # :59-65
    x = oracle.random_matrix(30, 22, 220)
    m = basic(x, 15)
    assert len(m.residual_history) == m.d
    h = m.residual_history
    assert all(h[k] <= h[k - 1] + 1e-12 for k in range(1, len(h)))


def test_T_rows_exact(cuda):                              # :67-74
    x = oracle.random_matrix(17, 12, 230)
    m = basic(x, 6)
    for k in range(m.d):
        assert np.abs(m.T[k] - x.T @ m.Y[:, k]).max() < 1e-13


def test_selected_distinct_in_range(cuda):                # :76-86
    x = oracle.random_matrix(26, 14, 240)
    m = basic(x, 10)
    assert len(m.selected) == m.d
    assert all(0 <= s < 14 for s in m.selected)
    assert len(set(m.selected)) == m.d


def test_certification(cuda):                             # :88-111 (identity weight)
    eps = 1e-5
    base = oracle.random_low_rank(40, 25, 6, 250)
    x = base / np.linalg.norm(base) + 1e-7 * oracle.random_matrix(40, 25, 251)
    m = basic(x, 25, eps)
    assert m.residual_history[-1] <= eps
    assert m.d < 25
    r = x - m.Y @ m.T
    assert np.sqrt((r * r).sum(0)).max() <= eps + 1e-10


def test_brute_force_projector(cuda):                     # :139-151
    for seed in (280, 281):
        x = oracle.random_matrix(50, 40, seed)
        m = basic(x, 20)
        y = m.Y
        brute = y @ np.linalg.solve(y.T @ y, y.T @ x)
        fast = y @ (y.T @ x)
        assert np.abs(brute - fast).max() < 1e-10
        assert np.abs(fast - m.Y @ m.T).max() < 1e-10


def test_start_column_control(cuda):                      # :153-169
    x = oracle.random_matrix(15, 10, 290)
    assert basic(x, 3, start_column=7).selected[0] == 7
    with pytest.raises(rbd.IndexOutOfRange):
        basic(x, 3, start_column=10)
    a = basic(x, 3, start_seed=42)
    b = basic(x, 3, start_seed=42)
    assert a.selected[0] == b.selected[0]
    assert 0 <= a.selected[0] < 10
    assert a.selected[0] == oracle.seeded_start(42, 10)   # same libstdc++ draw


def test_first_step_takes_start_column(cuda):             # :171-180
    x = oracle.random_matrix(12, 8, 300)
    for i in (0, 3, 7):
        m = basic(x, 1, start_column=i)
        xn = x[:, i] / np.linalg.norm(x[:, i])
        assert abs(abs(m.Y[:, 0] @ xn) - 1.0) < 1e-13


def test_input_gating(cuda):                              # :182-206
    x = oracle.random_matrix(10, 6, 310)
    with pytest.raises(rbd.DegenerateInput):
        basic(np.zeros((4, 3)), 2)
    with pytest.raises(rbd.InvalidArgument):
        basic(x, 0)
    with pytest.raises(rbd.InvalidArgument):
        basic(x, 7)
    with pytest.raises(rbd.InvalidArgument):
        basic(x, 2, -1.0)
    xn = x.copy()
    xn[3, 2] = np.nan
    with pytest.raises(rbd.InvalidArgument):
        basic(xn, 2)
    xi = x.copy()
    xi[0, 0] = np.inf
    with pytest.raises(rbd.InvalidArgument):
        basic(xi, 2)
    with pytest.raises(rbd.IncompatibleWeight):
        rbd.decompose(x, d_max=2, diag=np.ones(9))
    z = x.copy()
    z[:, 0] = 0.0
    with pytest.raises(rbd.DegenerateInput):
        basic(z, 2, breakdown_tol=1e-12)
    with pytest.raises(rbd.InvalidArgument):
        basic(np.zeros((0, 3)), 1)


def test_reorthogonalization_krylov(cuda):                # :231-244
    m_ = 60
    t = np.arange(1, m_ + 1) / m_
    x = np.stack([t ** j for j in range(8)], axis=1)
    m = basic(x, 8, reorthogonalize=True, breakdown_tol=1e-12)
    assert orthonormality_defect(m.Y) < 1e-12


def test_project_reconstruct(cuda):                       # :246-256
    x = oracle.random_matrix(18, 12, 320)
    m = basic(x, 5)
    c = oracle.random_matrix(5, 1, 321)[:, 0]
    v = m.reconstruct(c)
    assert np.abs(m.project(v) - c).max() < 1e-12
    with pytest.raises(rbd.DimensionMismatch):
        m.project(np.ones(17))
    with pytest.raises(rbd.DimensionMismatch):
        m.reconstruct(np.ones(4))


def test_mgs_project_device(cuda):                        # :274-289 + SPEC.md:67-71
    import torch
    x = oracle.random_matrix(10, 3, 340)
    y = (x[:, 0] / np.linalg.norm(x[:, 0]))[:, None]
    T = lambda a: torch.as_tensor(np.asfortranarray(a), device=cuda)
    res = rbd.mgs_project(T(x[:, 1]), T(y), 1e-12)
    assert res is not None
    xi, nrm = res
    xi = xi.cpu().numpy()
    assert abs(np.linalg.norm(xi) - 1.0) < 1e-14
    assert abs(xi @ y[:, 0]) < 1e-13
    manual = x[:, 1] - (y[:, 0] @ x[:, 1]) * y[:, 0]
    assert abs(nrm - np.linalg.norm(manual)) <= 1e-12 * np.linalg.norm(manual)
    assert rbd.mgs_project(T(3.7 * y[:, 0]), T(y), 1e-10) is None
    e1 = np.array([1.0, 0.0, 0.0])
    xi, nrm = rbd.mgs_project(T(e1), None, 1e-12)
    assert np.allclose(xi.cpu().numpy(), e1) and nrm == 1.0
    assert rbd.mgs_project(T(e1), T(e1[:, None]), 1e-12) is None
    xi, nrm = rbd.mgs_project(T(np.array([1.0, 1.0, 0.0])), T(e1[:, None]), 1e-12)
    assert np.allclose(xi.cpu().numpy(), [0.0, 1.0, 0.0]) and abs(nrm - 1.0) < 1e-15


def test_repeated_column(cuda):
    c = np.array([1.0, -2.0, 0.5, 3.0])
    x = np.stack([c, c, c], axis=1)
    m = basic(x, 3, 1e-12)
    assert m.d == 1
    assert np.allclose(m.T[0], np.linalg.norm(c) * np.ones(3), rtol=1e-15, atol=1e-14)


# ---------------- ports of proj/tests/python/test_smoke.py ----------------

def test_python_smoke_low_rank(cuda):                     # test_smoke.py:7-16
    rng = np.random.default_rng(7)
    x = rng.normal(size=(40, 6)) @ rng.normal(size=(6, 30))
    model = rbd.decompose(x, d_max=30, eps_r=1e-10)
    assert model.d == 6
    assert np.max(np.abs(x - model.Y @ model.T)) < 1e-9
    gram = model.Y.T @ model.Y
    assert np.max(np.abs(gram - np.eye(model.d))) < 1e-10
    hist = model.residual_history
    assert all(b <= a + 1e-12 for a, b in zip(hist, hist[1:]))
    assert len(model.selected) == model.d


def test_python_smoke_roundtrip(cuda):                    # test_smoke.py:19-28
    rng = np.random.default_rng(8)
    x = rng.normal(size=(25, 10))
    model = rbd.decompose(x, d_max=10)
    v = x[:, 3]
    c = model.project(v)
    assert c.shape == (model.d,)
    assert np.linalg.norm(model.reconstruct(c) - v) < 1e-9
    assert np.allclose(model.compress(), model.Y @ model.T)


def test_python_smoke_errors_typed(cuda):                 # test_smoke.py:82-84
    with pytest.raises(rbd.RbdError):
        rbd.decompose(np.zeros((4, 3)), d_max=2)


# ---------------- acceptance.cpp criteria 1, 2, 4 ----------------

@pytest.mark.parametrize("name,expected", [("rank1", 1), ("rank2", 2), ("rank3", 2)])
def test_acceptance1_exact_rank(cuda, name, expected):   # :95-138 (+ README aliasing note)
    x = oracle.gen_grid_matrix(name, 201)
    m = basic(x, 10, 1e-10)
    assert m.d == expected
    assert np.sqrt(((x - m.Y @ m.T) ** 2).sum(0)).max() < 1e-8


def test_acceptance2_composite(cuda):                     # :142-177, test_output.txt:13
    x = oracle.gen_grid_matrix("composite", 1001)
    g = basic(x, 22)
    r = oracle.decompose(x, 22)
    assert g.d == 22
    err = np.abs(x - g.Y @ g.T).max()
    assert err < 1e-5
    assert 1e-9 < err < 1e-7          # recorded 7.496e-09 in the reference run
    compare(g, r, x)


def test_acceptance4_invariants(cuda):                    # :242-297
    battery = [oracle.random_matrix(50, 50, 1), oracle.random_matrix(50, 30, 2),
               oracle.random_matrix(30, 50, 3),
               oracle.random_matrix(40, 8, 4) @ oracle.random_matrix(8, 40, 5),
               oracle.gen_grid_matrix("composite", 50)]
    for x in battery:
        d_max = min(25, x.shape[1])
        m = basic(x, d_max, 1e-6)
        assert orthonormality_defect(m.Y) < 1e-10
        h = m.residual_history
        assert all(h[k] <= h[k - 1] + 1e-12 for k in range(1, len(h)))
        if h[-1] <= 1e-6:
            assert np.sqrt(((x - m.Y @ m.T) ** 2).sum(0)).max() <= 1e-6 + 1e-10
        again = basic(x, d_max, 1e-6)
        assert np.array_equal(again.Y, m.Y) and np.array_equal(again.T, m.T)
        assert again.selected == m.selected
        y = m.Y
        brute = y @ np.linalg.solve(y.T @ y, y.T @ x)
        assert np.abs(brute - m.Y @ m.T).max() < 1e-10
        compare(m, oracle.decompose(x, d_max, 1e-6), x)


def test_host_entry_pinned_outputs_stream_y_from_the_loop(cuda):
    # large enough for page-locked host outputs (api._host_outputs): the
    # persistent loop writes Y into them directly; must equal the device entry
    rng = np.random.default_rng(21)
    x = np.asfortranarray(rng.standard_normal((8192, 300)))
    h = rbd.decompose(x, d_max=150)
    import torch
    dv = rbd.decompose(torch.from_numpy(x).cuda(), d_max=150)
    assert h.selected == dv.selected
    np.testing.assert_array_equal(h.Y, dv.Y.cpu().numpy())
    np.testing.assert_array_equal(h.T, dv.T.cpu().numpy())


def test_host_many_pipelined_equals_single_calls(cuda):
    """rbd_decompose_host_many (upload of matrix i+1 during matrix i's loop,
    two device X buffers) gives every matrix the bits of a single host call;
    pinned and pageable inputs, fp64 and fp32 storage."""
    import torch
    m, n, d = 9000, 260, 40
    xs = []
    for i in range(5):
        a = oracle.random_matrix(m, n, 500 + i)
        if i % 2 == 0:   # page-locked
            t = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
            t.copy_(torch.from_numpy(np.ascontiguousarray(a.T)))
            a = t.numpy().T
        xs.append(a)
    many = rbd.decompose_many(xs, d_max=d, eps_r=1e-9)
    assert len(many) == len(xs)
    for x, g in zip(xs, many):
        s = rbd.decompose(np.asfortranarray(x), d_max=d, eps_r=1e-9)
        assert g.selected == s.selected and g.d == s.d
        assert np.array_equal(g.Y, s.Y) and np.array_equal(g.T, s.T)
        assert g.residual_history == s.residual_history
    xs32 = [np.asfortranarray(x, dtype=np.float32) for x in xs[:3]]
    many32 = rbd.decompose_many(xs32, d_max=d)
    for x, g in zip(xs32, many32):
        s = rbd.decompose(x, d_max=d)
        assert g.selected == s.selected and np.array_equal(g.Y, s.Y) and np.array_equal(g.T, s.T)
    assert rbd.decompose_many([], d_max=3) == []
    with pytest.raises(rbd.InvalidArgument):
        rbd.decompose_many([xs[0], xs[1][:, :10]], d_max=3)


def test_host_many_stops_at_a_failing_matrix(cuda):
    """A non-finite matrix in the middle of the sequence raises the reference's
    InvalidArgument (decompose.cpp:57); the uploads still in flight are drained
    and the context stays usable."""
    xs = [oracle.random_matrix(500, 30, 900 + i) for i in range(3)]
    xs[1] = xs[1].copy()
    xs[1][7, 3] = np.nan
    with pytest.raises(rbd.InvalidArgument):
        rbd.decompose_many(xs, d_max=5)
    ok = rbd.decompose_many([xs[0], xs[2]], d_max=5)
    assert [g.d for g in ok] == [5, 5]


def test_overflowing_column_norms_return_an_error_and_keep_the_context(cuda):
    """Finite entries near 1e160 overflow ||x_j||^2 to inf. The reference then
    has max_col_norm = inf, so breakdown_tol = inf (decompose.cpp:70-74) and the
    first mgs_project of a normal start column breaks down: DegenerateInput
    (:104-105) — the oracle's outcome below. The B200 path returns that error
    before its loop starts (no NaN partial can reach the loop's ready-flag
    protocol), and the context stays usable. (When the start column itself
    overflows, the reference divides by an infinite norm and returns zero basis
    vectors with an inf history; the B200 path returns the same error there.)"""
    import torch
    rng = np.random.default_rng(5)
    x = rng.standard_normal((64, 9))
    x[:, 5] = rng.choice([-1.0, 1.0], size=64) * 1e160
    with pytest.raises(oracle.OracleError) as ei:
        oracle.decompose(x, 4)
    assert ei.value.kind == "DegenerateInput"
    ctx = rbd.Context(0)
    with pytest.raises(rbd.DegenerateInput):
        rbd.decompose(x, d_max=4, ctx=ctx)
    with pytest.raises(rbd.DegenerateInput):
        rbd.decompose(x * 0 + 1e160, d_max=4, ctx=ctx)
    with pytest.raises(rbd.DegenerateInput):
        rbd.decompose(torch.as_tensor(x, device=cuda), d_max=4, ctx=ctx)
    # weighted: finite ||x_j||^2 but a_i * ||x_j||^2 overflows
    xw = rng.choice([-1.0, 1.0], size=(64, 9)) * 1e150
    with pytest.raises(rbd.InvalidArgument):
        rbd.decompose(xw, d_max=4, diag=np.full(64, 1e10), ctx=ctx)
    ok = rbd.decompose(oracle.random_matrix(30, 10, 7), d_max=5, ctx=ctx)
    r = oracle.decompose(oracle.random_matrix(30, 10, 7), 5)
    assert ok.selected == r.selected
    assert np.abs(ok.Y - r.Y).max() < 1e-12
    torch.cuda.synchronize()
