"""compress_matrix / batched reconstruct V = Y T on the FP64 tensor cores (SURVEY
§8(f3); decompose.cpp:119-125) against a float64 host product. Tolerance: the
fp64 dot-product bound d * eps * sum_k |Y_ik||T_kj| (any summation order)."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
import paper_1503_05947_b200 as rbd
from paper_1503_05947_b200._lib import check, load_library

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


def assert_product(V, Y, T):
    ref = Y @ T
    bound = Y.shape[1] * EPS * (np.abs(Y) @ np.abs(T)) + 1e-300
    assert np.all(np.abs(np.asarray(V) - ref) <= bound)


@pytest.mark.parametrize("m,n,d", [(32256, 2432, 400), (33, 17, 5), (4097, 130, 17), (64, 64, 64),
                                   (1000, 1, 3), (129, 65, 129)])
def test_device_compress_matches_fp64_product(cuda, m, n, d):
    rng = np.random.default_rng(m + n + d)
    x = rng.standard_normal((m, max(n, d)))
    model = rbd.decompose(torch.from_numpy(np.asfortranarray(x)).cuda(), d_max=d)
    V = model.compress()
    assert V.is_cuda and V.shape == (m, max(n, d))
    assert_product(V.cpu().numpy(), model.Y.cpu().numpy(), model.T.cpu().numpy())


def test_host_compress_and_reconstruct_batch(cuda):
    x = oracle.random_matrix(300, 80, 5)
    model = rbd.decompose(x, d_max=30)
    assert_product(model.compress(), model.Y, model.T)
    # reconstruct is the one-column case (decompose.cpp:119-123); consistent with project
    v = x[:, 7]
    c = model.project(v)
    np.testing.assert_allclose(model.reconstruct(c), model.Y @ c, rtol=0, atol=1e-12)


def test_odd_row_stride_takes_the_fallback(cuda):
    lib = load_library()
    ctx = rbd.default_context(0)
    m, d, n = 40, 6, 9                      # odd ldt -> unaligned rows of T
    Y = torch.randn(d, m, dtype=torch.float64, device="cuda").t()
    T = torch.randn(d, n, dtype=torch.float64, device="cuda")
    V = torch.empty(n, m, dtype=torch.float64, device="cuda").t()
    torch.cuda.synchronize()
    check(lib.rbd_compress_device(ctx.handle, C.c_void_p(Y.data_ptr()), m, d, m,
                                  C.c_void_p(T.data_ptr()), n, n, C.c_void_p(V.data_ptr()), m))
    ctx.synchronize()
    assert_product(V.cpu().numpy(), Y.cpu().numpy(), T.cpu().numpy())
