"""RBD1 model container through the C ABI (rbd_model_write /
rbd_model_read_header / rbd_model_read) on host buffers (no GPU needed): byte
parity with the oracle's restatement of io.cpp:533-570 and the reference's own
container tests (proj/tests/test_io.cpp:273-345, python/test_smoke.py:47-48)."""
import os

import numpy as np
import pytest

import oracle
import paper_1503_05947_b200 as rbd
from paper_1503_05947_b200._lib import Result


def host_model(om, kind=0, diag=None):
    res = Result()
    res.d = om.d
    return rbd.Model(np.asfortranarray(om.Y), np.ascontiguousarray(om.T), om.d, om.selected,
                     om.residual_history, res, None, kind, diag)


@pytest.fixture
def scratch(tmp_path):
    return tmp_path


def models():
    x = oracle.random_matrix(12, 9, 1040)                        # test_io.cpp:273-285
    ident = oracle.decompose(x, 5, 1e-9)
    dg = oracle.random_positive(12, 1041)
    diag = oracle.decompose(x, 5, 1e-9, diag=dg)
    return [("identity", host_model(ident)), ("diagonal", host_model(diag, 1, dg)),
            ("sparse_external", host_model(ident, 2))]


@pytest.mark.parametrize("which", [0, 1, 2])
def test_round_trip_bit_exact_every_tag(scratch, which):        # test_io.cpp:273-311
    name, model = models()[which]
    p = scratch / "model.rbd"
    model.save(p, eps_r=1e-9)
    raw = p.read_bytes()
    assert raw == oracle.model_bytes(model.Y, model.T, 1e-9, model.residual_history,
                                     model.weight_kind, model.diag)
    back, eps = rbd.load(p)
    assert np.array_equal(back.Y, model.Y)
    assert np.array_equal(back.T, model.T)
    assert back.d == model.d
    assert back.residual_history == model.residual_history
    assert eps == 1e-9
    assert back.weight_kind == model.weight_kind
    if model.weight_kind == 1:
        assert np.array_equal(back.diag, model.diag)
    m, d, n = model.Y.shape[0], model.d, model.T.shape[1]
    expect = 29 + 8 * (m * d + d * n + 1 + d) + (8 * m if model.weight_kind == 1 else 0)
    assert os.path.getsize(p) == expect
    assert back.selected == []                                   # not stored (io.hpp:56)
    assert not os.path.exists(str(p) + ".tmp")


def test_corrupted_files_are_rejected(scratch):                  # test_io.cpp:313-332
    x = oracle.random_matrix(6, 5, 1050)
    model = host_model(oracle.decompose(x, 3))
    p = scratch / "corrupt.rbd"
    model.save(p, 0.0)
    raw = p.read_bytes()
    p.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(rbd.ParseError, match="bad magic"):
        rbd.load(p)
    p.write_bytes(raw[:-8])                                      # truncated payload
    with pytest.raises(rbd.ParseError, match="size does not match"):
        rbd.load(p)
    bad = bytearray(raw)
    bad[28] = 9
    p.write_bytes(bytes(bad))
    with pytest.raises(rbd.ParseError, match="unknown weight tag"):
        rbd.load(p)
    bad = bytearray(raw)
    bad[20:28] = (6).to_bytes(8, "little")                       # d > n
    p.write_bytes(bytes(bad))
    with pytest.raises(rbd.ParseError, match="implausible model dimensions"):
        rbd.load(p)
    p.write_bytes(raw[:10])
    with pytest.raises(rbd.ParseError) as e:
        rbd.load(p)
    assert str(e.value).startswith(str(p) + ":0: ")              # ParseError(path, 0, what)


def test_missing_file_raises_io_error(scratch):                  # test_io.cpp:341-345
    with pytest.raises(rbd.IoError):
        rbd.load(scratch / "nope.rbd")


def test_unwritable_destination_raises_io_error(scratch):
    model = host_model(oracle.decompose(oracle.random_matrix(6, 5, 1), 2))
    with pytest.raises(rbd.IoError):
        model.save(scratch / "no_such_dir" / "m.rbd")


def test_overwrite_is_atomic(scratch):                           # test_io.cpp:334-340
    p = scratch / "overwrite.rbd"
    a = host_model(oracle.decompose(oracle.random_matrix(8, 6, 2), 3))
    b = host_model(oracle.decompose(oracle.random_matrix(10, 7, 3), 4))
    a.save(p)
    b.save(p)
    back, _ = rbd.load(p)
    assert np.array_equal(back.Y, b.Y) and np.array_equal(back.T, b.T)
    assert not os.path.exists(str(p) + ".tmp")


def test_python_smoke_save_load(scratch):                        # test_smoke.py:47-48
    x = oracle.random_matrix(20, 15, 102)
    dg = np.linspace(0.5, 2.5, 20)                               # acceptance.cpp:439
    model = host_model(oracle.decompose(x, 6, 1e-8, diag=dg), 1, dg)
    p = scratch / "m.rbd"
    model.save(p, eps_r=1e-8)
    back, eps_r = rbd.load(p)
    assert eps_r == 1e-8
    assert np.array_equal(back.Y, model.Y) and np.array_equal(back.diag, dg)
    # the parsed payload equals the oracle's reading of the same bytes
    Y, T, e, h, tag, diag = oracle.parse_model(p.read_bytes())
    assert np.array_equal(Y, back.Y) and np.array_equal(T, back.T) and tag == 1


def test_inconsistent_shapes_rejected(scratch):
    model = host_model(oracle.decompose(oracle.random_matrix(6, 5, 4), 3))
    model.residual_history = model.residual_history[:2]
    bad = rbd.Model(model.Y, model.T[:2], 3, [], model.residual_history, Result(), None)
    with pytest.raises(rbd.RbdError):
        bad.save(scratch / "x.rbd")
