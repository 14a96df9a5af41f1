"""Breakdown fidelity near the noise floor (decompose.cpp:29-30,70-74).

The greedy loop stops when the orthogonalised candidate's norm ||w|| drops
below breakdown_tol = max(eps_R or cfg.breakdown_tol, max_j ||x_j|| sqrt(m) eps 16).
A rank-r matrix plus noise of standard deviation sigma leaves residual columns
of norm ~ sigma sqrt(m) after r steps, so sweeping sigma across
tol / sqrt(m) moves the stop from d = r (breakdown) to d = d_max. At every
sigma the B200 loop must end where the oracle ends, with the same breakdown
flag — except when the oracle's ||w|| at the deciding step lies within the
rounding band of two backward-stable orthogonalisations of the same column
(64 eps ||x_j|| sqrt(k+1)), where either decision is admissible (the analogue
of the near-tie rule for selections)."""
import numpy as np
import pytest

import oracle
import paper_1503_05947_b200 as rbd
from parity import compare, running_residuals

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


def low_rank_plus_noise(m, n, r, sigma, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, r))
    B = rng.standard_normal((r, n))
    X = A @ B / np.sqrt(r) + sigma * rng.standard_normal((m, n))
    return np.asfortranarray(X)


def deciding_norm(X, ref, k):
    """Oracle ||w|| of the candidate examined at step k (accepted or broken down)."""
    if k < ref.d:
        j = ref.selected[k]
    else:
        _, rs = running_residuals(X, ref.T)
        j = int(np.argmax(rs[k - 1])) if k > 0 else 0
    res = oracle.mgs_project(X[:, j], ref.Y[:, :k] if k else None, 0.0)
    return (res[1] if res is not None else 0.0), float(np.linalg.norm(X[:, j]))


@pytest.mark.parametrize("m,n,r", [(300, 60, 8), (5000, 40, 5)])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_noise_sweep_across_the_floor(cuda, m, n, r, seed):
    base = low_rank_plus_noise(m, n, r, 0.0, seed)
    floor_sigma = np.sqrt((base * base).sum(0)).max() * EPS * 16.0   # tol / sqrt(m)
    ds = []
    ambiguous = 0
    for f in (0.25, 0.5, 0.8, 1.0, 1.25, 2.0, 4.0):
        X = low_rank_plus_noise(m, n, r, f * floor_sigma, seed)
        g = rbd.decompose(X, d_max=n)
        ref = oracle.decompose(X, n)
        ref_breakdown = ref.d < n                      # eps_R = 0: only a breakdown stops early
        assert g.selected[:min(g.d, ref.d)] == ref.selected[:min(g.d, ref.d)]
        if g.d != ref.d:
            k = min(g.d, ref.d)
            nrm, xn = deciding_norm(X, ref, k)
            band = 64.0 * EPS * xn * np.sqrt(k + 1)
            assert abs(nrm - g.result.breakdown_tol) <= band, (
                f"sigma={f}*floor: d gpu {g.d} vs oracle {ref.d}; oracle ||w|| {nrm:.6e}, "
                f"tol {g.result.breakdown_tol:.6e} (band {band:.1e})")
            ambiguous += 1
        else:
            assert bool(g.result.breakdown) == ref_breakdown, f"sigma={f}*floor"
            compare(g, ref, X, require_same_d=True)
        ds.append(ref.d)
    assert ds[0] == r and ds[-1] == n          # the sweep crosses the floor
    assert ambiguous <= 1


def test_guard_band_recompute_path(cuda):
    """breakdown_tol set to the oracle's own ||w|| at step k puts the decision
    inside the guard band, where the loop recomputes ||w1 - Y p|| from the
    materialised column (rbd_device.cuh: exact_wnorm2) instead of
    sqrt(||w1||^2 - ||p||^2). Either outcome is admissible there; the run must
    stop at step k or k+1 with parity on the common prefix."""
    X = low_rank_plus_noise(400, 30, 6, 1e-3, 11)
    ref_full = oracle.decompose(X, 30, breakdown_tol=0.0)
    for k in (3, 7, 12):
        nrm, _ = deciding_norm(X, ref_full, k)
        g = rbd.decompose(X, d_max=30, breakdown_tol=nrm)
        ref = oracle.decompose(X, 30, breakdown_tol=nrm)
        assert g.d in (k, k + 1) and ref.d in (k, k + 1)
        compare(g, ref, X, require_same_d=False)
