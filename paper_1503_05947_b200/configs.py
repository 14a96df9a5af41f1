"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is involved; every input is generated from a fixed seed.
Choices for the under-specified parts of BASELINE.json (recorded in the bench
JSON ``config`` and in DESIGN.md §Workloads):
  * "N(0, v)" noise is read as VARIANCE v (sigma = sqrt(v)).
  * C1 "tol=1e-3 relative" -> absolute eps_R = 1e-3 * max_j ||x_j|| (the
    reference's eps_R is absolute, decompose.hpp:27).
  * C1 frames are 192x168 flattened column-major (pixel = row + 192*col).
  * C2/C3/C4 use eps_R = 0 (reference default) so the noise-floor breakdown
    tolerance governs (decompose.cpp:70-74).
Randomness comes from numpy (C0, C1 parameters) or a seeded torch.Generator
(C2-C4 on the GPU); generation is plumbing, not the measured path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    m: int
    n: int
    d_max: int
    eps_rel: float      # eps_R = eps_rel * max_j ||x_j|| (C1) ...
    eps_abs: float      # ... or absolute eps_R
    seed: int
    describe: str


C0 = Workload("C0-cpu-ref", 1024, 512, 64, 0.0, 1e-6, 0,
              "X=U diag(2^(-i/4)) V^T + N(0,1e-6), rank 64, U/V QR-orthonormalised Gaussian")
C1 = Workload("C1-image-like", 32256, 2432, 400, 1e-3, 0.0, 1,
              "192x168 frames, 8-32 Gaussian blobs/col (sigma 4-40px, amp 0-255) + U[0,2) noise, clip [0,255]")
C2 = Workload("C2-tall", 1 << 20, 4096, 512, 0.0, 0.0, 2,
              "low-rank+noise, rank 1024, s_i=(1+i)^-1.5, N(0,1e-8)")
C3 = Workload("C3-sharded", 1 << 18, 1 << 16, 1024, 0.0, 0.0, 3,
              "low-rank+noise, rank 2048, s_i=exp(-i/256), N(0,1e-10); 8192-col shards/GPU")
C4 = Workload("C4-out-of-sample", 1 << 16, 8192, 512, 0.0, 0.0, 4,
              "RBD on rank-512 (s_i=2^(-i/4)) + N(0,1e-6); then 262144 new cols in batches of 16384")

WORKLOADS = {w.name: w for w in (C0, C1, C2, C3, C4)}
FRAME = (192, 168)


def c0_matrix(m: int = 1024, n: int = 512, rank: int = 64, seed: int = 0,
              noise_var: float = 1e-6) -> np.ndarray:
    """BASELINE config 0: X = U diag(s) V^T + noise (numpy, column-major)."""
    rng = np.random.default_rng(seed)
    U = np.linalg.qr(rng.standard_normal((m, rank)))[0]
    V = np.linalg.qr(rng.standard_normal((n, rank)))[0]
    s = 2.0 ** (-np.arange(rank) / 4.0)
    X = (U * s) @ V.T + np.sqrt(noise_var) * rng.standard_normal((m, n))
    return np.asfortranarray(X)


def blob_params(n: int, seed: int = 1, frame=FRAME):
    """Per-column blob parameters for C1 (numpy, seeded)."""
    rng = np.random.default_rng(seed)
    H, W = frame
    counts = rng.integers(8, 33, size=n)          # 8..32 blobs
    kmax = 32
    cy = rng.uniform(0, H, size=(n, kmax))
    cx = rng.uniform(0, W, size=(n, kmax))
    sig = rng.uniform(4.0, 40.0, size=(n, kmax))
    amp = rng.uniform(0.0, 255.0, size=(n, kmax))
    mask = np.arange(kmax)[None, :] < counts[:, None]
    amp = amp * mask
    return cy, cx, sig, amp


def c1_matrix(n: int = 2432, seed: int = 1, device="cpu", frame=FRAME, batch: int = 64):
    """BASELINE config 1 (image-like), returned as a column-major torch tensor
    (m x n view of an (n, m) contiguous buffer) on ``device``."""
    import torch

    H, W = frame
    m = H * W
    cy, cx, sig, amp = blob_params(n, seed, frame)
    noise_rng = np.random.default_rng(seed + 1000)
    out = torch.empty((n, m), dtype=torch.float64, device=device)
    rr = torch.arange(H, dtype=torch.float64, device=device)
    cc = torch.arange(W, dtype=torch.float64, device=device)
    # pixel p = row + H*col (column-major flattening of an H x W frame)
    R = rr.repeat(W)                      # row of pixel p
    Cc = cc.repeat_interleave(H)          # col of pixel p
    for j0 in range(0, n, batch):
        j1 = min(n, j0 + batch)
        t = lambda a: torch.as_tensor(a[j0:j1], dtype=torch.float64, device=device)
        y0, x0, s, a = t(cy), t(cx), t(sig), t(amp)
        dy = R[None, None, :] - y0[:, :, None]
        dx = Cc[None, None, :] - x0[:, :, None]
        g = torch.exp(-(dy * dy + dx * dx) / (2.0 * s[:, :, None] ** 2))
        val = (a[:, :, None] * g).sum(dim=1)
        noise = torch.as_tensor(noise_rng.uniform(0.0, 2.0, size=(j1 - j0, m)), device=device)
        out[j0:j1] = torch.clamp(val + noise, 0.0, 255.0)
    return out.t()  # (m, n), stride (1, m)


def low_rank_matrix_torch(m: int, n: int, rank: int, s, noise_var: float, seed: int,
                          device="cuda"):
    """X = U diag(s) V^T + N(0, noise_var), U/V QR-orthonormalised Gaussian, on
    ``device`` (column-major m x n view). Used for C2, C3, C4."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    U = torch.linalg.qr(torch.randn(m, rank, dtype=torch.float64, device=device, generator=g))[0]
    V = torch.linalg.qr(torch.randn(n, rank, dtype=torch.float64, device=device, generator=g))[0]
    sv = torch.as_tensor(np.asarray(s, dtype=np.float64), device=device)
    Xt = torch.empty((n, m), dtype=torch.float64, device=device)  # X^T row-major = X col-major
    for j0 in range(0, n, 1024):
        j1 = min(n, j0 + 1024)
        blk = (V[j0:j1] * sv) @ U.t()
        blk += float(np.sqrt(noise_var)) * torch.randn(blk.shape, dtype=torch.float64,
                                                       device=device, generator=g)
        Xt[j0:j1] = blk
    del U, V
    return Xt.t()


def spectrum(name: str, rank: int):
    i = np.arange(rank, dtype=np.float64)
    if name == "C2":
        return (1.0 + i) ** -1.5
    if name == "C3":
        return np.exp(-i / 256.0)
    return 2.0 ** (-i / 4.0)  # C0 / C4 ("as in config 0")


def eps_for(w: Workload, max_col_norm: float) -> float:
    return w.eps_abs if w.eps_rel == 0.0 else w.eps_rel * max_col_norm


def low_rank_shard_torch(m: int, n: int, rank: int, s, noise_var: float, seed: int,
                         col_offset: int, n_local: int, device="cuda", block: int = 1024):
    """Columns [col_offset, col_offset + n_local) of the same X as
    low_rank_matrix_torch-style generation, identical for any sharding:
    U, V from one generator (seed), noise per 1024-column block from a
    generator keyed by (seed, block)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    U = torch.linalg.qr(torch.randn(m, rank, dtype=torch.float64, device=device, generator=g))[0]
    V = torch.linalg.qr(torch.randn(n, rank, dtype=torch.float64, device=device, generator=g))[0]
    sv = torch.as_tensor(np.asarray(s, dtype=np.float64), device=device)
    Xt = torch.empty((n_local, m), dtype=torch.float64, device=device)
    sigma = float(np.sqrt(noise_var))
    gn = torch.Generator(device=device)
    for b0 in range((col_offset // block) * block, col_offset + n_local, block):
        lo, hi = max(b0, col_offset), min(b0 + block, col_offset + n_local)
        gn.manual_seed(seed * 1000003 + b0 // block)
        noise = torch.randn((min(block, n - b0), m), dtype=torch.float64, device=device, generator=gn)
        blk = (V[lo:hi] * sv) @ U.t()
        blk += sigma * noise[lo - b0:hi - b0]
        Xt[lo - col_offset:hi - col_offset] = blk
    del U, V
    return Xt.t()


# ---- config 4: the RBD stage and the out-of-sample stream ----
C4_RANK = 512
C4_BATCH = 16384
C4_NEW_COLUMNS = 262144


def c4_stage_matrix(device="cuda"):
    """The C4 RBD stage (65536 x 8192, rank 512, s_i = 2^(-i/4), N(0,1e-6)) — the
    same X as ``low_rank_matrix_torch`` builds for bench / tools."""
    w = C4
    return low_rank_matrix_torch(w.m, w.n, C4_RANK, spectrum("C4", C4_RANK), 1e-6, w.seed,
                                 device=device)


def c4_basis(device="cuda"):
    """U (m x 512) and s of the C4 low-rank model (the first draws of the seed-4
    generator, as in low_rank_matrix_torch)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(C4.seed)
    U = torch.linalg.qr(torch.randn(C4.m, C4_RANK, dtype=torch.float64, device=device,
                                    generator=g))[0]
    s = torch.as_tensor(spectrum("C4", C4_RANK), device=device)
    return U, s


def c4_new_batch(U, s, b: int, batch: int = C4_BATCH, device="cuda"):
    """Out-of-sample batch b of C4: x = U diag(s) g + e with g ~ N(0, I)/sqrt(8192)
    (the stage's column distribution) and e ~ N(0, 1e-6); column-major m x batch.
    Each batch has its own generator keyed by (seed, b), so any batch can be
    regenerated alone."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(C4.seed * 1000003 + 7919 + b)
    coef = torch.randn(batch, C4_RANK, dtype=torch.float64, device=device, generator=g)
    coef /= float(np.sqrt(C4.n))
    Xt = (coef * s) @ U.t()                                   # batch x m == X col-major
    Xt += 1e-3 * torch.randn(Xt.shape, dtype=torch.float64, device=device, generator=g)
    return Xt.t()
