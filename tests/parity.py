"""Parity protocol between the B200 path and the CPU oracle.

* selected: equal step by step, except where the oracle's top-two residual gap
  at that step is within tau * max_j col_sq_j (a near tie, either pick is
  admissible); comparison of Y/T/history stops at the first admissible
  divergence, or, given `rerun`, continues over all steps on a B200 re-run
  forced onto the oracle's selection (rbd_set_forced_selection).
* Y:        ||y_k^gpu - y_k^ref||_2 <= tol_k,  tol_k = tol + 64 eps kappa_k
            (tol = 1e-10 fp64). kappa_k = ||x_{j_k}|| / ||w_k|| is the factor by
            which step k amplifies roundoff: y_k = w_k/||w_k|| with
            w_k = x_{j_k} - Y Y'x_{j_k}, so any two backward-stable
            orthogonalisations differ by O(eps kappa_k) in y_k. For
            well-conditioned steps tol_k == 1e-10 to within 1%.
* T:        |T_kj^gpu - T_kj^ref|  <= tol_k * ||x_j||
* history:  |e_k^2(gpu) - e_k^2(ref)| <= 2 sum_{l<=k} tol_l * max_j col_sq_j (the
            running residual bookkeeping col_sq - sum t^2 cancels, so the error
            scales with col_sq, not with e_k^2; cf. acceptance.cpp:223,
            test_workspace.cpp:91)
* diagonal weight: selection follows the A-norm residual
  e2_j = ||x_j - Y T_j||_A^2, so near ties and the history bound use those
  residuals (computed directly from the oracle's Y and T) and max col_sq_A;
  kappa_k stays Euclidean (the orthogonalisation is Euclidean).
"""
from __future__ import annotations

import numpy as np


def running_residuals(X: np.ndarray, T: np.ndarray, col_sq=None):
    """Oracle-side residual_sq after each step (workspace.cpp:52-53). col_sq
    (||x_j||^2) may be given instead of X (X streamed in blocks)."""
    if col_sq is None:
        col_sq = np.einsum("ij,ij->j", X, X)
    r = np.asarray(col_sq, dtype=np.float64).copy()
    out = []
    for k in range(T.shape[0]):
        r = np.maximum(r - T[k] * T[k], 0.0)
        out.append(r.copy())
    return col_sq, out


def weighted_residuals(X: np.ndarray, Y: np.ndarray, T: np.ndarray, diag: np.ndarray):
    """Oracle-side A-norm residuals after each step (workspace.cpp:84-99 evaluated
    directly: ||x_j - Y_k T_k[:, j]||_A^2)."""
    col_sq = np.einsum("ij,i,ij->j", X, diag, X)
    out = []
    for k in range(T.shape[0]):
        R = X - Y[:, : k + 1] @ T[: k + 1]
        out.append(np.maximum(np.einsum("ij,i,ij->j", R, diag, R), 0.0))
    return col_sq, out


def top2_gap(r: np.ndarray) -> float:
    if r.size < 2:
        return np.inf
    a = np.partition(r, -2)[-2:]
    return float(abs(a[1] - a[0]))


def compare(gpu, ref, X, tol: float = 1e-10, tau: float = 1e-12, require_same_d: bool = True,
            diag=None, rerun=None, col_sq=None):
    """Returns the number of steps compared; raises AssertionError on mismatch.

    rerun: optional callable(selected) -> gpu model. After an admissible
    divergence the B200 loop is re-run on the oracle's selection (forced-selection
    mode, rbd_set_forced_selection) and compared over all steps.
    col_sq: ||x_j||^2 in place of X (identity weight; X too large for the host)."""
    if col_sq is None:
        X = np.asarray(X, dtype=np.float64)
    gY = np.asarray(gpu.Y.cpu() if hasattr(gpu.Y, "cpu") else gpu.Y)
    gT = np.asarray(gpu.T.cpu() if hasattr(gpu.T, "cpu") else gpu.T)
    col_sq, rsteps = running_residuals(X, ref.T, col_sq)
    colnorm = np.sqrt(col_sq)
    if diag is None:
        sel_sq, ssteps = col_sq, rsteps
    else:
        sel_sq, ssteps = weighted_residuals(X, ref.Y, ref.T, np.asarray(diag, dtype=np.float64))
    max_colsq = float(sel_sq.max())
    d_cmp = min(gpu.d, ref.d)
    upto = d_cmp
    for k in range(d_cmp):
        if gpu.selected[k] != ref.selected[k]:
            assert k > 0, f"start column differs: {gpu.selected[0]} vs {ref.selected[0]}"
            gap = top2_gap(ssteps[k - 1])
            assert gap <= tau * max_colsq, (
                f"selected diverges at step {k}: gpu {gpu.selected[k]} ref {ref.selected[k]}, "
                f"top-two gap {gap:.3e} > {tau * max_colsq:.3e}")
            upto = k
            break
    if upto < d_cmp and rerun is not None:
        forced = rerun(list(ref.selected))
        assert list(forced.selected[:ref.d]) == list(ref.selected[:forced.d])
        return compare(forced, ref, X, tol, tau, require_same_d, diag, col_sq=col_sq)
    if upto == d_cmp and require_same_d:
        assert gpu.d == ref.d, f"d differs: gpu {gpu.d} ref {ref.d}"
    tols = step_tolerances(ref, col_sq, rsteps, tol)
    for k in range(upto):
        dy = float(np.linalg.norm(gY[:, k] - ref.Y[:, k]))
        assert dy <= tols[k], f"Y column {k}: ||dy|| = {dy:.3e} > {tols[k]:.3e}"
    if upto:
        dT = np.abs(gT[:upto] - ref.T[:upto]) / np.maximum(colnorm, 1e-300)[None, :]
        for k in range(upto):
            assert dT[k].max() <= tols[k], (
                f"T row {k}: max |dT|/||x_j|| = {dT[k].max():.3e} > {tols[k]:.3e}")
        gh = np.asarray(gpu.residual_history[:upto])
        rh = np.asarray(ref.residual_history[:upto])
        bound = 2.0 * np.cumsum(tols[:upto]) * max_colsq
        dh = np.abs(gh * gh - rh * rh)
        assert np.all(dh <= bound), f"history mismatch: {dh.max():.3e} (bound {bound.max():.3e})"
    return upto


EPS = np.finfo(np.float64).eps


def step_tolerances(ref, col_sq, rsteps, tol):
    """tol_k = tol + 64 eps kappa_k with kappa_k = ||x_j|| / ||w_k|| (oracle side)."""
    out = []
    for k in range(ref.d):
        j = ref.selected[k]
        r_before = col_sq[j] if k == 0 else rsteps[k - 1][j]
        kappa = np.sqrt(col_sq[j] / max(r_before, 1e-300))
        out.append(tol + 64.0 * EPS * kappa)
    return np.asarray(out)


def orthonormality_defect(Y) -> float:
    Y = np.asarray(Y)
    return float(np.abs(Y.T @ Y - np.eye(Y.shape[1])).max()) if Y.shape[1] else 0.0
