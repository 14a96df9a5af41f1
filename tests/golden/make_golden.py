"""Generates tests/golden/*.npz from the CPU oracle (oracle/rbd_oracle.cpp).

The reference cannot be compiled here (Eigen 3.4 absent), so
these fixtures are the oracle's outputs on fixed inputs; the oracle itself is
pinned to the reference's recorded values by tests/test_oracle_pins.py. The
fixtures freeze the checker: tests/test_golden.py recomputes them bit-exactly
on CPU, and the GPU tests compare the B200 path against them.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1503_05947_b200 import configs  # noqa: E402

CASES = {
    # name: (input builder, d_max, eps_R, kwargs)
    "c0": (lambda: configs.c0_matrix(), 64, 1e-6, {}),
    "composite201": (lambda: oracle.gen_grid_matrix("composite", 201), 22, 0.0, {}),
    "random50x40_s280": (lambda: oracle.random_matrix(50, 40, 280), 20, 0.0, {}),
    "lowrank40x30_r5": (lambda: oracle.random_low_rank(40, 30, 5, 210), 30, 0.0, {}),
    "krylov60x8_reorth": (lambda: np.stack([(np.arange(1, 61) / 60) ** j for j in range(8)], 1),
                          8, 0.0, {"reorthogonalize": True, "breakdown_tol": 1e-12}),
    "seeded_start_15x10": (lambda: oracle.random_matrix(15, 10, 290), 3, 0.0, {"start_seed": 42}),
}


def compute(name):
    build, d_max, eps, kw = CASES[name]
    X = np.asfortranarray(build())
    r = oracle.decompose(X, d_max, eps, **kw)
    return X, r


def main():
    for name in CASES:
        X, r = compute(name)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), selected=np.asarray(r.selected),
                            history=np.asarray(r.residual_history), Y=r.Y, T=r.T, d=r.d,
                            x_checksum=np.float64(np.sum(X * np.arange(1, X.size + 1).reshape(X.shape, order="F"))))
        print(name, r.d)


if __name__ == "__main__":
    main()
