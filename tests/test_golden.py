"""Golden fixtures (tests/golden/make_golden.py): the oracle reproduces them
bit-exactly (CPU), and the B200 path matches them under the parity protocol
(GPU)."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import make_golden  # noqa: E402

from parity import compare  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("name", sorted(make_golden.CASES))
def test_oracle_reproduces_golden(name):
    g = load(name)
    X, r = make_golden.compute(name)
    chk = np.sum(X * np.arange(1, X.size + 1).reshape(X.shape, order="F"))
    assert chk == g["x_checksum"], "fixture input changed"
    assert r.d == int(g["d"])
    assert r.selected == list(g["selected"])
    assert np.array_equal(np.asarray(r.residual_history), g["history"])
    assert np.array_equal(r.Y, g["Y"]) and np.array_equal(r.T, g["T"])


class _Ref:
    def __init__(self, g):
        self.Y, self.T, self.d = g["Y"], g["T"], int(g["d"])
        self.selected = [int(s) for s in g["selected"]]
        self.residual_history = [float(h) for h in g["history"]]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(make_golden.CASES))
def test_gpu_matches_golden(cuda, name):
    import paper_1503_05947_b200 as rbd
    g = load(name)
    build, d_max, eps, kw = make_golden.CASES[name]
    X = np.asfortranarray(build())
    m = rbd.decompose(X, d_max=d_max, eps_r=eps, **kw)
    compare(m, _Ref(g), X)
