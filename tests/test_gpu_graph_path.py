"""The per-phase fallback path of the greedy loop (a CUDA graph of G steps of
K4 / K2 / K3 kernels; used for d_max above the persistent kernel's 4096-column
coefficient cache, or with RBD_PATH=graph): parity with the oracle, and a
decomposition past 4096 steps checked through its full-size properties."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1503_05947_b200 as rbd
from paper_1503_05947_b200 import configs
from parity import compare, orthonormality_defect

pytestmark = pytest.mark.gpu


@pytest.fixture
def graph_ctx(cuda):
    os.environ["RBD_PATH"] = "graph"        # read when a context is created
    try:
        ctx = rbd.Context(0)
    finally:
        del os.environ["RBD_PATH"]
    yield ctx
    ctx.close()


@pytest.mark.parametrize("shape", [(1024, 512, 64), (333, 80, 40), (4097, 33, 20)])
def test_graph_path_parity(graph_ctx, shape):
    m, n, d = shape
    x = configs.c0_matrix() if shape == (1024, 512, 64) else oracle.random_matrix(m, n, m + n)
    g = rbd.decompose(x, d_max=d, eps_r=1e-6 if shape[0] == 1024 else 0.0, ctx=graph_ctx)
    r = oracle.decompose(x, d, 1e-6 if shape[0] == 1024 else 0.0)
    assert compare(g, r, x) == r.d


def test_graph_path_reorth_and_seeded_start(graph_ctx):
    # noise well above the residual bookkeeping's cancellation level (~eps * |x|^2):
    # at 1e-9 the post-rank argmax is decided by rounding (it can re-pick a
    # selected column, which then breaks down) and any summation order is "right"
    x = oracle.random_low_rank(300, 90, 12, 5) + 1e-4 * oracle.random_matrix(300, 90, 6)
    g = rbd.decompose(x, d_max=40, reorthogonalize=True, start_seed=99, ctx=graph_ctx)
    r = oracle.decompose(x, 40, reorthogonalize=True, start_seed=99)
    compare(g, r, x)


def test_more_than_4096_steps(cuda):
    # d_max > 4096 selects the graph path automatically; full-rank Gaussian input
    m, n, d = 4608, 4352, 4200
    gen = torch.Generator(device="cuda").manual_seed(8)
    X = torch.randn(n, m, generator=gen, device="cuda", dtype=torch.float64).t()
    g = rbd.decompose(X, d_max=d)
    assert g.d == d
    Y = g.Y
    assert float((Y.t() @ Y - torch.eye(d, device="cuda", dtype=torch.float64)).abs().max()) < 1e-10
    cols = torch.arange(0, n, 97, device="cuda")
    err = (g.T[:, cols] - Y.t() @ X[:, cols]).abs().max() / X[:, cols].norm(dim=0).max()
    assert float(err) < 1e-12
    assert len(set(g.selected)) == d
    h = np.asarray(g.residual_history)
    assert np.all(np.diff(h) <= 1e-12 * h[0])
