"""Device-resident models (rbd_model_t) and the out-of-sample
entries on them: project (decompose.cpp:113-117), reconstruct (:119-123), the
pipelined batch stream of config 4 (rbd_project_host_many[_f32]) and
read_model straight into HBM (io.cpp:574-622)."""
import time

import numpy as np
import pytest

import oracle
import paper_1503_05947_b200 as rbd

pytestmark = pytest.mark.gpu


def pinned(a, dtype=np.float64):
    import torch
    a = np.asarray(a, dtype=dtype)
    t = torch.empty((a.shape[1], a.shape[0]), dtype=torch.float64 if dtype == np.float64
                    else torch.float32, pin_memory=True)
    t.copy_(torch.from_numpy(np.ascontiguousarray(a.T)))
    return t.numpy().T


def test_resident_project_matches_device_kernel_and_oracle(cuda):
    import torch
    x = oracle.random_matrix(3000, 60, 41)
    g = rbd.decompose(x, d_max=25)
    rm = rbd.ResidentModel.from_model(g)
    assert (rm.m, rm.n, rm.d) == (3000, 60, 25)
    xn = oracle.random_matrix(3000, 37, 42)
    Tn, err = rm.project(xn)
    Td, ed = rbd.project_batch(torch.as_tensor(g.Y, device=cuda),
                               torch.as_tensor(np.asfortranarray(xn), device=cuda))
    assert np.array_equal(Tn, Td.cpu().numpy()) and np.array_equal(err, ed.cpu().numpy())
    Tr, er = oracle.project_batch(g.Y, xn)
    sc = np.sqrt((xn * xn).sum(0))
    assert (np.abs(Tn - Tr) / sc).max() < 1e-13
    assert (np.abs(err - er) / sc ** 2).max() < 1e-12
    # the Model API routes host models through the resident copy
    c = g.project(xn[:, 5])
    assert np.array_equal(c, Tn[:, 5])
    assert g._resident is not None
    v = g.reconstruct(c)
    assert np.abs(v - g.Y @ c).max() < 1e-12
    with pytest.raises(rbd.DimensionMismatch):
        rm.project(np.ones(2999))
    with pytest.raises(rbd.DimensionMismatch):
        rm.reconstruct(np.ones(24))


def test_project_stream_equals_single_batches(cuda):
    x = oracle.random_matrix(4096, 80, 51)
    g = rbd.decompose(x, d_max=64)
    rm = g.resident()
    batches = [pinned(oracle.random_matrix(4096, 300, 60 + i)) for i in range(5)]
    outs = rm.project_many(batches)
    for b, (T, e) in zip(batches, outs):
        T1, e1 = rm.project(b)
        assert np.array_equal(T, T1) and np.array_equal(e, e1)
    # fp32 mode: the model's fp32 copy of Y on tcgen05 (K6) — same bits as
    # project_batch_f32 on the same fp32 operands, and 1e-4 of the fp64 oracle
    import torch
    b32 = [pinned(b, np.float32) for b in batches[:3]]
    outs32 = rm.project_many(b32, f32=True)
    Y32 = torch.as_tensor(np.asfortranarray(g.Y.astype(np.float32)), device=cuda)
    for b, (T, e) in zip(b32, outs32):
        Tk, ek = rbd.project_batch_f32(Y32, torch.as_tensor(np.asfortranarray(b), device=cuda))
        assert np.array_equal(T, Tk.cpu().numpy()) and np.array_equal(e, ek.cpu().numpy())
        Tr, er = oracle.project_batch(g.Y.astype(np.float32).astype(np.float64),
                                      b.astype(np.float64))
        sc = np.sqrt((b.astype(np.float64) ** 2).sum(0))
        assert (np.abs(T - Tr) / sc).max() < 1e-4
    # pageable inputs still give the same results (no overlap)
    pg = [np.asfortranarray(np.array(b)) for b in batches[:2]]
    for b, (T, e) in zip(pg, rm.project_many(pg)):
        assert np.array_equal(T, rm.project(b)[0])
    assert rm.project_many([]) == []
    with pytest.raises(rbd.InvalidArgument):
        rm.project_many([batches[0], batches[1][:, :10]])


def test_resident_load_from_file(cuda, tmp_path):
    x = oracle.random_matrix(500, 40, 71)
    w = oracle.random_positive(500, 72)
    g = rbd.decompose(x, d_max=12, diag=w)
    p = tmp_path / "m.rbd"
    g.save(p, eps_r=0.5)
    rm = rbd.ResidentModel.load(p)
    assert (rm.m, rm.n, rm.d, rm.weight_kind, rm.eps_r) == (500, 40, 12, 1, 0.5)
    Y, T = rm.device_arrays()
    assert np.array_equal(Y.cpu().numpy(), g.Y) and np.array_equal(T.cpu().numpy(), g.T)
    assert np.array_equal(rm.history(), np.asarray(g.residual_history))
    v = x[:, 3]
    assert np.array_equal(rm.project(v)[0][:, 0], g.project(v))
    # a corrupt diagonal (WeightSpec::diagonal rejects non-positive values on read)
    raw = bytearray(p.read_bytes())
    raw[-8:] = np.float64(-1.0).tobytes()
    bad = tmp_path / "bad.rbd"
    bad.write_bytes(bytes(raw))
    with pytest.raises(rbd.InvalidArgument):
        rbd.ResidentModel.load(bad)
    with pytest.raises(rbd.InvalidArgument):
        rbd.load(bad)


def test_per_vector_project_on_c4_sized_basis_uploads_nothing_per_call(cuda):
    """1,024 per-vector project calls (classify.cpp:22-23, main.cpp:149-158) on a
    65,536 x 512 basis: the 256 MiB Y stays in HBM, each call moves one vector
    (an upload of Y per call alone would take >= 4.6 ms at PCIe rates)."""
    import torch
    m, d = 65536, 512
    gen = torch.Generator(device=cuda)
    gen.manual_seed(3)
    Yd = torch.linalg.qr(torch.randn(m, d, dtype=torch.float64, device=cuda, generator=gen))[0]
    Y = np.asfortranarray(Yd.cpu().numpy())
    from paper_1503_05947_b200._lib import Result
    model = rbd.Model(Y, np.zeros((d, d)), d, list(range(d)), [0.0] * d, Result(),
                      rbd.default_context(0))
    vs = np.random.default_rng(0).standard_normal((m, 1024))
    model.project(vs[:, 0])                        # creates the resident copy
    t0 = time.perf_counter()
    cs = [model.project(vs[:, j]) for j in range(1024)]
    dt = time.perf_counter() - t0
    ref = Y.T @ vs
    assert max(float(np.abs(c - ref[:, j]).max()) for j, c in enumerate(cs)) < 1e-11
    assert dt / 1024 < 3e-3, f"{dt / 1024 * 1e3:.2f} ms per project call"
