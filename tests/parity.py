"""Parity protocol between the B200 path and the CPU oracle.

* selected: equal step by step, except where the oracle's top-two residual gap
  at that step is within tau * max_j col_sq_j (a near tie, either pick is
  admissible); comparison of Y/T/history stops at the first admissible
  divergence.
* Y:        ||y_k^gpu - y_k^ref||_2 <= tol                    (tol = 1e-10, fp64)
* T:        |T_kj^gpu - T_kj^ref|  <= tol * ||x_j||
* history:  |e_k^2(gpu) - e_k^2(ref)| <= tol * max_j col_sq_j  (the running
            residual bookkeeping col_sq - sum t^2 cancels, so the error scales
            with col_sq, not with e_k^2; cf. acceptance.cpp:223, test_workspace.cpp:91)
"""
from __future__ import annotations

import numpy as np


def running_residuals(X: np.ndarray, T: np.ndarray):
    """Oracle-side residual_sq after each step (workspace.cpp:52-53)."""
    col_sq = np.einsum("ij,ij->j", X, X)
    r = col_sq.copy()
    out = []
    for k in range(T.shape[0]):
        r = np.maximum(r - T[k] * T[k], 0.0)
        out.append(r.copy())
    return col_sq, out


def top2_gap(r: np.ndarray) -> float:
    if r.size < 2:
        return np.inf
    a = np.partition(r, -2)[-2:]
    return float(abs(a[1] - a[0]))


def compare(gpu, ref, X, tol: float = 1e-10, tau: float = 1e-12, require_same_d: bool = True):
    """Returns the number of steps compared; raises AssertionError on mismatch."""
    X = np.asarray(X, dtype=np.float64)
    gY = np.asarray(gpu.Y.cpu() if hasattr(gpu.Y, "cpu") else gpu.Y)
    gT = np.asarray(gpu.T.cpu() if hasattr(gpu.T, "cpu") else gpu.T)
    col_sq, rsteps = running_residuals(X, ref.T)
    max_colsq = float(col_sq.max())
    colnorm = np.sqrt(col_sq)
    d_cmp = min(gpu.d, ref.d)
    upto = d_cmp
    for k in range(d_cmp):
        if gpu.selected[k] != ref.selected[k]:
            assert k > 0, f"start column differs: {gpu.selected[0]} vs {ref.selected[0]}"
            gap = top2_gap(rsteps[k - 1])
            assert gap <= tau * max_colsq, (
                f"selected diverges at step {k}: gpu {gpu.selected[k]} ref {ref.selected[k]}, "
                f"top-two gap {gap:.3e} > {tau * max_colsq:.3e}")
            upto = k
            break
    if upto == d_cmp and require_same_d:
        assert gpu.d == ref.d, f"d differs: gpu {gpu.d} ref {ref.d}"
    for k in range(upto):
        dy = float(np.linalg.norm(gY[:, k] - ref.Y[:, k]))
        assert dy <= tol, f"Y column {k}: ||dy|| = {dy:.3e} > {tol}"
    if upto:
        dT = np.abs(gT[:upto] - ref.T[:upto])
        ratio = (dT / np.maximum(colnorm, 1e-300)[None, :]).max()
        assert ratio <= tol, f"T mismatch: max |dT|/||x_j|| = {ratio:.3e} > {tol}"
        gh = np.asarray(gpu.residual_history[:upto])
        rh = np.asarray(ref.residual_history[:upto])
        dh = np.abs(gh * gh - rh * rh).max()
        assert dh <= tol * max_colsq, f"history mismatch: {dh:.3e} > {tol * max_colsq:.3e}"
    return upto


def orthonormality_defect(Y) -> float:
    Y = np.asarray(Y)
    return float(np.abs(Y.T @ Y - np.eye(Y.shape[1])).max()) if Y.shape[1] else 0.0
