"""CPU checks of the oracle pieces the config-scale parity tests rely on
(tests/test_gpu_configs.py): the column-block restatement of the greedy loop,
the single-pass option and the tiled batch projection all give the bits of the
whole-matrix, per-vector oracle (decompose.cpp:53-117, workspace.cpp:50-53)."""
import ctypes as C

import numpy as np
import pytest

import oracle


@pytest.mark.parametrize("m,n,d,blocks", [(3000, 70, 40, [(0, 25), (25, 30), (55, 15)]),
                                          (517, 33, 33, [(0, 1), (1, 31), (32, 1)]),
                                          (64, 9, 9, [(0, 9)])])
def test_blocked_and_single_pass_loops_equal_the_oracle(m, n, d, blocks):
    X = oracle.random_matrix(m, n, 4000 + m)
    r = oracle.decompose(X, d, nthreads=3)
    r1 = oracle.decompose(X, d, nthreads=2, x_passes=1)
    rb = oracle.decompose_blocked(lambda b: X[:, blocks[b][0]:blocks[b][0] + blocks[b][1]],
                                  blocks, m, n, d, nthreads=2)
    for o in (r1, rb):
        assert o.selected == r.selected and o.d == r.d
        assert np.array_equal(o.Y, r.Y) and np.array_equal(o.T, r.T)
        assert o.residual_history == r.residual_history
    assert np.array_equal(rb.col_sq, oracle.column_sq(X, 2))
    assert r.t_loop_s >= 0.0 and r.t_init_s >= 0.0


def test_blocked_loop_prefix_and_errors():
    X = oracle.random_matrix(200, 12, 77)
    blocks = [(0, 5), (5, 7)]
    get = lambda b: X[:, blocks[b][0]:blocks[b][0] + blocks[b][1]]  # noqa: E731
    rb = oracle.decompose_blocked(get, blocks, 200, 12, 10, max_steps=4,
                                  get_column=lambda j: X[:, j])
    r = oracle.decompose(X, 10, max_steps=4)
    assert rb.selected == r.selected and np.array_equal(rb.T, r.T)
    Xn = X.copy()
    Xn[3, 7] = np.inf
    with pytest.raises(oracle.OracleError) as e:
        oracle.decompose_blocked(lambda b: Xn[:, blocks[b][0]:blocks[b][0] + blocks[b][1]],
                                 blocks, 200, 12, 10)
    assert e.value.kind == "InvalidArgument"
    with pytest.raises(oracle.OracleError) as e:
        oracle.decompose_blocked(get, blocks, 200, 12, 13)
    assert e.value.kind == "InvalidArgument"
    Z = np.zeros((200, 12))
    with pytest.raises(oracle.OracleError) as e:
        oracle.decompose_blocked(lambda b: Z[:, :blocks[b][1]], blocks, 200, 12, 3)
    assert e.value.kind == "DegenerateInput"


@pytest.mark.parametrize("m,d,N", [(1003, 13, 70), (4096, 64, 33), (7, 2, 3), (20000, 130, 45),
                                   (5000, 1, 1)])
def test_tiled_batch_projection_equals_per_vector_project(m, d, N):
    rng = np.random.default_rng(m + d)
    Y = np.asfortranarray(rng.standard_normal((m, d)))
    X = np.asfortranarray(rng.standard_normal((m, N)))
    Tn, err = oracle.project_batch(Y, X, nthreads=4)
    L = oracle.lib()
    L.orc_project.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
    for j in range(N):
        c = np.zeros(d)
        L.orc_project(oracle._p(Y), m, d, oracle._p(np.ascontiguousarray(X[:, j])), oracle._p(c))
        assert np.array_equal(c, Tn[:, j])
        e = float(oracle.column_sq(X[:, j:j + 1])[0] - (c * c).sum())
        assert abs(max(e, 0.0) - err[j]) <= 1e-12 * float((X[:, j] ** 2).sum())
