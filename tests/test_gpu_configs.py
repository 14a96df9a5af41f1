"""Oracle parity at the sizes of BASELINE.json's configurations 2-4 (north star:
"oracle-matching RBD on all five configs"; C0 and C1 are in
test_gpu_decompose.py). Each test runs the B200 path through the C ABI on the
configuration's seeded synthetic X, compares a prefix (or all) of its greedy
steps with the CPU oracle under the parity protocol of tests/parity.py
(SURVEY.md §8(c)), and checks size-independent properties of the WHOLE run:
orthonormal Y, T == Y'X on sampled columns, monotone history, distinct
selections (test_decompose.cpp:42-86, acceptance.cpp:265-269).

* C2-tall (1,048,576 x 4,096, d = 512): the first 64 steps against the
  threaded oracle on the host copy of X (34 GB).
* C3-sharded on one GPU (262,144 x 65,536, d = 1024; 128 GiB of X): the first
  8 steps against the oracle run over 4,096-column blocks streamed from HBM
  (oracle.decompose_blocked), so X never has to sit in host memory at once.
* C4 RBD stage (65,536 x 8,192, d = 512): all 512 steps.
* C4 out-of-sample: one 16,384-column batch, fp64 (K5, DMMA) against
  oracle.project_batch (per-vector project, decompose.cpp:113-117, plus the
  Eq. 3 indicator, workspace.cpp:88-97) at 1e-10, and the fp32 mode (K6,
  tcgen05 3xTF32) against the oracle on the fp32-rounded inputs at 1e-4.
"""
import gc
import os

import numpy as np
import pytest

import oracle
import paper_1503_05947_b200 as rbd
from paper_1503_05947_b200 import configs
from parity import compare

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

NCPU = os.cpu_count() or 1


@pytest.fixture
def fresh_gpu(cuda):
    import torch
    gc.collect()
    torch.cuda.empty_cache()
    yield cuda
    gc.collect()
    torch.cuda.empty_cache()


class _Prefix:
    """The first d steps of a B200 model, as host arrays, for parity.compare."""

    def __init__(self, g, d):
        self.Y = g.Y[:, :d].cpu().numpy()
        self.T = g.T[:d].cpu().numpy()
        self.d = d
        self.selected = list(g.selected[:d])
        self.residual_history = list(g.residual_history[:d])


def full_run_properties(g, Xd, sample: int = 512, seed: int = 0):
    """Size-independent checks of a whole device run (test_decompose.cpp:42-86)."""
    import torch
    Y, T = g.Y, g.T
    G = Y.t() @ Y
    G.diagonal().sub_(1.0)
    defect = float(G.abs().max())
    assert defect < 1e-10, f"orthonormality defect {defect:.3e}"
    del G
    n = Xd.shape[1]
    idx = torch.as_tensor(np.sort(np.random.default_rng(seed).choice(n, min(sample, n),
                                                                     replace=False)),
                          device=Xd.device)
    Xs = Xd[:, idx]
    Td = Y.t() @ Xs
    norms = Xs.norm(dim=0)
    dT = float(((Td - T[:, idx]).abs() / norms).max())
    assert dT < 1e-12, f"T != Y'X on sampled columns: {dT:.3e}"
    h = np.asarray(g.residual_history)
    assert np.all(h[1:] <= h[:-1] + 1e-12 * float(norms.max())), "history not monotone"
    assert len(set(g.selected)) == g.d, "selected columns repeat"
    return defect, dT


# ---------------- C2-tall ----------------

def test_c2_parity_64_steps_and_full_properties(fresh_gpu):
    import torch
    cuda = fresh_gpu
    w = configs.C2
    Xd = configs.low_rank_matrix_torch(w.m, w.n, 1024, configs.spectrum("C2", 1024), 1e-8,
                                       w.seed, device=cuda)
    g = rbd.decompose(Xd, d_max=w.d_max)
    assert g.d == w.d_max
    full_run_properties(g, Xd)
    Xh = torch.empty((w.n, w.m), dtype=torch.float64, pin_memory=True)
    Xh.copy_(Xd.t())
    del Xd
    X = Xh.numpy().T
    steps = 64
    r = oracle.decompose(X, w.d_max, nthreads=NCPU, max_steps=steps, x_passes=1)
    assert r.d == steps
    assert compare(_Prefix(g, steps), r, None, col_sq=oracle.column_sq(X, NCPU)) == steps


# ---------------- C3 on one GPU (128 GiB) ----------------

def test_c3_first_steps_blocked_oracle_and_full_properties(fresh_gpu):
    import torch
    cuda = fresh_gpu
    w = configs.C3
    Xd = configs.low_rank_shard_torch(w.m, w.n, 2048, configs.spectrum("C3", 2048), 1e-10,
                                      w.seed, 0, w.n, device=cuda)
    g = rbd.decompose(Xd, d_max=w.d_max)
    assert g.d == w.d_max
    full_run_properties(g, Xd)
    Xt = Xd.t()                                     # n x m row-major == X column-major
    B = 4096
    blocks = [(o, min(B, w.n - o)) for o in range(0, w.n, B)]
    hbuf = torch.empty((B, w.m), dtype=torch.float64, pin_memory=True)

    def get_block(b):
        o, nb = blocks[b]
        hbuf[:nb].copy_(Xt[o:o + nb])
        return hbuf[:nb].numpy().T

    steps = 8
    r = oracle.decompose_blocked(get_block, blocks, w.m, w.n, w.d_max, nthreads=NCPU,
                                 max_steps=steps, get_column=lambda j: Xt[j].cpu().numpy())
    assert r.d == steps
    assert compare(_Prefix(g, steps), r, None, col_sq=r.col_sq) == steps


# ---------------- C4: RBD stage + out-of-sample compression ----------------

@pytest.fixture(scope="module")
def c4_stage(cuda):
    import torch
    gc.collect()
    torch.cuda.empty_cache()
    Xd = configs.c4_stage_matrix(cuda)
    g = rbd.decompose(Xd, d_max=configs.C4.d_max)
    yield Xd, g
    del Xd, g
    gc.collect()
    torch.cuda.empty_cache()


def test_c4_rbd_stage_full_parity(c4_stage):
    Xd, g = c4_stage
    w = configs.C4
    assert g.d == w.d_max
    full_run_properties(g, Xd)
    X = np.asfortranarray(Xd.cpu().numpy())
    r = oracle.decompose(X, w.d_max, nthreads=NCPU, x_passes=1)

    def rerun(sel):
        return _Prefix(rbd.decompose(Xd, d_max=w.d_max, forced_selection=sel), len(sel))
    assert compare(_Prefix(g, g.d), r, X, rerun=rerun) == w.d_max


def _c4_batch(cuda):
    U, s = configs.c4_basis(cuda)
    Xn = configs.c4_new_batch(U, s, 0, device=cuda)
    del U
    return Xn


def test_c4_out_of_sample_batch_fp64(c4_stage, cuda):
    Xd, g = c4_stage
    Y = g.Y.t().contiguous().t()
    Xn = _c4_batch(cuda)
    assert tuple(Xn.shape) == (configs.C4.m, configs.C4_BATCH)
    Tn, err = rbd.project_batch(Y, Xn)
    Tr, er = oracle.project_batch(Y.cpu().numpy(), Xn.cpu().numpy(), nthreads=NCPU)
    xx = oracle.column_sq(Xn.cpu().numpy(), NCPU)
    dT = float((np.abs(Tn.cpu().numpy() - Tr) / np.sqrt(xx)).max())
    dE = float((np.abs(err.cpu().numpy() - er) / xx).max())
    assert dT < 1e-10, dT          # north_star fp64 parity
    assert dE < 1e-10, dE


def test_c4_out_of_sample_batch_fp32(c4_stage, cuda):
    import torch
    Xd, g = c4_stage
    Y32 = g.Y.to(torch.float32).t().contiguous().t()
    X32 = _c4_batch(cuda).to(torch.float32).t().contiguous().t()
    Tn, err = rbd.project_batch_f32(Y32, X32)
    Yr = Y32.double().cpu().numpy()
    Xr = X32.double().cpu().numpy()
    Tr, er = oracle.project_batch(Yr, Xr, nthreads=NCPU)
    xx = oracle.column_sq(Xr, NCPU)
    dT = float((np.abs(Tn.double().cpu().numpy() - Tr) / np.sqrt(xx)).max())
    dE = float((np.abs(err.cpu().numpy() - er) / xx).max())
    assert dT < 1e-4, dT           # north_star fp32-mode parity
    assert dE < 1e-4, dE
