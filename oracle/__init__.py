"""TEST INFRASTRUCTURE ONLY — the CPU oracle of the RBD greedy loop.

ctypes wrapper over ``oracle/build/liborc.so`` (oracle/rbd_oracle.cpp, a
plain-loop restatement of /root/reference/proj/src/decompose.cpp:12-125 and
workspace.cpp:9-125, identity path). Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs may import this package; the product package
never does.

Parity pinning: the reference cannot be compiled here (Eigen 3.4 absent), so
the restatement is pinned by the reference's own known-answer values and
property tests, ported in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liborc.so")

ORC_OK = 0
ORC_INCOMPATIBLE_WEIGHT = 2
ERRORS = {1: "InvalidArgument", 2: "IncompatibleWeight", 3: "DegenerateInput",
          4: "IndexOutOfRange", 5: "DimensionMismatch"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            import subprocess
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        L = C.CDLL(LIB_PATH)
        P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
        L.orc_last_error.restype = C.c_char_p
        L.orc_decompose_steps.argtypes = [P, I64, I64, I64, I64, D, I, I64, C.c_uint64, I, D, I, I64,
                                          P, P, P, P, P]
        L.orc_decompose_steps.restype = I
        L.orc_decompose_ex.argtypes = [P, I64, I64, I64, I64, D, I, I64, C.c_uint64, I, D, I, I64,
                                       I, P, P, P, P, P, P, P]
        L.orc_decompose_ex.restype = I
        L.orc_column_pass.argtypes = [P, I64, I64, I64, I, P, P, P]
        L.orc_gemv_t.argtypes = [P, I64, I64, I64, P, P, I]
        L.orc_mgs_project.argtypes = [P, I64, P, I64, I64, D, I, P, P]
        L.orc_mgs_project.restype = I
        L.orc_ws_init.argtypes = [P, I64, I64, I64]
        L.orc_ws_init.restype = P
        L.orc_ws_free.argtypes = [P]
        L.orc_ws_extend.argtypes = [P, P]
        L.orc_ws_d.argtypes = [P]
        L.orc_ws_d.restype = I64
        L.orc_ws_col_sq.argtypes = [P, P]
        L.orc_ws_residual.argtypes = [P, P]
        L.orc_ws_yax_row.argtypes = [P, I64, P]
        L.orc_ws_error_sq.argtypes = [P, I64, P, I64, P]
        L.orc_ws_error_sq.restype = I
        L.orc_ws_scan.argtypes = [P, P, P]
        L.orc_project.argtypes = [P, I64, I64, P, P]
        L.orc_project.restype = None
        L.orc_reconstruct.argtypes = [P, I64, I64, P, P]
        L.orc_project_batch.argtypes = [P, I64, I64, P, I64, I64, I, P, P]
        L.orc_random_matrix.argtypes = [I64, I64, C.c_uint64, P]
        L.orc_random_low_rank.argtypes = [I64, I64, I64, C.c_uint64, P]
        L.orc_gen_grid_matrix.argtypes = [I, I64, P]
        L.orc_gen_grid_matrix.restype = I
        L.orc_acceptance3_count.restype = I64
        L.orc_seeded_start.argtypes = [C.c_uint64, I64]
        L.orc_seeded_start.restype = I64
        L.orc_decompose_diag.argtypes = [P, I64, I64, I64, P, I64, I64, D, I, I64, C.c_uint64, I,
                                         D, I64, P, P, P, P, P]
        L.orc_decompose_diag.restype = I
        L.orc_ws_init_diag.argtypes = [P, I64, I64, I64, P, I64]
        L.orc_ws_init_diag.restype = P
        L.orc_ws_scan_T.argtypes = [P, P, P, P]
        L.orc_ws_scan_T.restype = I
        L.orc_ws_yay.argtypes = [P, P]
        L.orc_ws_yay.restype = I
        L.orc_random_positive.argtypes = [I64, C.c_uint64, P]
        L.orc_predict_batch.argtypes = [P, I64, I64, P, I64, P, I64, I, P, P]
        L.orc_gen_labeled_blobs.argtypes = [I, I, I, D, C.c_uint64, P, P]
        L.orc_gen_labeled_blobs.restype = I
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class OracleModel:
    Y: np.ndarray                 # m x d
    T: np.ndarray                 # d x n
    selected: List[int]
    residual_history: List[float]
    d: int = 0
    t_init_s: float = 0.0         # validation + workspace_init wall time
    t_loop_s: float = 0.0         # greedy loop wall time


def decompose(x, d_max: int, eps_r: float = 0.0, start_column: int = 0,
              start_seed: Optional[int] = None, reorthogonalize: bool = False,
              breakdown_tol: float = -1.0, nthreads: int = 1,
              max_steps: Optional[int] = None, diag=None, x_passes: int = 2) -> OracleModel:
    """rbd::decompose restated (decompose.cpp:53-111); diag = WeightSpec::diagonal.

    x_passes=2 keeps the reference's two X passes per step (decompose.cpp:93,
    workspace.cpp:51); 1 reuses the first pass (same bits, half the time)."""
    xa = np.asfortranarray(np.asarray(x, dtype=np.float64))
    m, n = xa.shape if xa.ndim == 2 else (0, 0)
    cap = max(1, min(int(d_max), max(n, 1)))
    Y = np.zeros((m, cap), order="F")
    T = np.zeros((cap, max(n, 1)))
    sel = np.zeros(cap, dtype=np.int64)
    hist = np.zeros(cap)
    d = C.c_int64(0)
    steps = int(max_steps if max_steps is not None else 2**62)
    seed = int(start_seed or 0) & 0xFFFFFFFFFFFFFFFF
    kind = 1 if start_seed is not None else 0
    ti, tl = C.c_double(), C.c_double()
    if diag is not None:
        dg = np.ascontiguousarray(np.asarray(diag, dtype=np.float64).reshape(-1))
        rc = lib().orc_decompose_diag(
            _p(xa), m, n, max(m, 1), _p(dg) if dg.size else None, dg.size, int(d_max),
            float(eps_r), kind, int(start_column), seed, 1 if reorthogonalize else 0,
            float(breakdown_tol), steps, _p(Y), _p(T), _p(sel), _p(hist), C.byref(d))
    else:
        rc = lib().orc_decompose_ex(
            _p(xa), m, n, max(m, 1), int(d_max), float(eps_r), kind, int(start_column), seed,
            1 if reorthogonalize else 0, float(breakdown_tol), int(nthreads), steps,
            int(x_passes), _p(Y), _p(T), _p(sel), _p(hist), C.byref(d), C.byref(ti), C.byref(tl))
    if rc != ORC_OK:
        raise OracleError(rc, lib().orc_last_error().decode())
    k = d.value
    return OracleModel(Y[:, :k].copy(order="F"), T[:k, :n].copy(), [int(s) for s in sel[:k]],
                       [float(h) for h in hist[:k]], k, ti.value, tl.value)


def decompose_blocked(get_block, blocks, m: int, n: int, d_max: int, eps_r: float = 0.0,
                      start_column: int = 0, nthreads: int = 1,
                      max_steps: Optional[int] = None, get_column=None) -> OracleModel:
    """rbd::decompose (decompose.cpp:53-111, identity weight, fixed start
    column, default config) over an X that is only available in column blocks:
    ``blocks`` is a list of (col_offset, n_cols) covering [0, n) in order and
    ``get_block(i)`` returns block i as an m x n_cols column-major float64
    array (``get_column(j)``, optional, column j alone). Each greedy step streams every block once (the reference's two
    passes per step compute identical values, so the second is reused). Used
    for config 3 (128 GiB of X) by the parity tests; the arithmetic is the
    whole-matrix oracle's (per-column dot8 sums, the same mgs_project)."""
    L = lib()
    steps = int(max_steps if max_steps is not None else 2**62)
    # ---- validation (decompose.cpp:56-64) and workspace_init (workspace.cpp:21-23) ----
    if m < 1 or n < 1:
        raise OracleError(1, "decompose: matrix must be non-empty")
    sq = np.zeros(n)
    fin, zero = True, True
    for b, (o, nb) in enumerate(blocks):
        xb = get_block(b)
        f, z = C.c_int(), C.c_int()
        L.orc_column_pass(_p(xb), m, nb, xb.strides[1] // 8, int(nthreads),
                          _p(sq[o:o + nb]), C.byref(f), C.byref(z))
        fin, zero = fin and bool(f.value), zero and bool(z.value)
    if not fin:
        raise OracleError(1, "decompose: matrix has non-finite entries")
    if d_max < 1 or d_max > n:
        raise OracleError(1, "decompose: d_max must satisfy 1 <= d_max <= n")
    if not eps_r >= 0.0:
        raise OracleError(1, "decompose: eps_R must be >= 0")
    if zero:
        raise OracleError(3, "decompose: zero matrix, no basis can be built")
    max_col_norm = float(np.sqrt(sq).max())                                 # :70
    noise_floor = max_col_norm * np.sqrt(float(m)) * np.finfo(np.float64).eps * 16.0
    breakdown_tol = max(eps_r, noise_floor)                                  # :73-74
    col_sq = np.maximum(sq, 0.0)                                             # workspace.cpp:37
    residual = col_sq.copy()
    if not 0 <= start_column < n:
        raise OracleError(4, "start column index out of range")
    i = int(start_column)
    cap = min(int(d_max), steps)
    Y = np.zeros((m, max(cap, 1)), order="F")
    T = np.zeros((max(cap, 1), n))
    sel, hist = [], []
    d = 0
    e_cur = np.inf

    def column(j):
        if get_column is not None:
            return np.ascontiguousarray(get_column(j), dtype=np.float64)
        for b, (o, nb) in enumerate(blocks):
            if o <= j < o + nb:
                return np.ascontiguousarray(get_block(b)[:, j - o])
        raise IndexError(j)

    xi = np.zeros(m)
    nrm = C.c_double()
    while d < d_max and e_cur > eps_r and d < steps:                         # :87
        v = column(i)
        ok = L.orc_mgs_project(_p(v), m, _p(Y), d, m, float(breakdown_tol), 0, _p(xi),
                               C.byref(nrm))
        if not ok:
            break                                                            # :90
        Y[:, d] = xi                                                         # :92
        for b, (o, nb) in enumerate(blocks):                                 # :93
            xb = get_block(b)
            L.orc_gemv_t(_p(xb), m, nb, xb.strides[1] // 8, _p(xi), _p(T[d, o:o + nb]),
                         int(nthreads))
        sel.append(i)
        residual = np.maximum(residual - T[d] * T[d], 0.0)                   # workspace.cpp:52-53
        d += 1
        arg = int(np.argmax(residual))            # strict '>' scan from j = 0 (workspace.cpp:107-113)
        best = float(residual[arg])
        e_cur = float(np.sqrt(best if best > 0.0 else 0.0))
        hist.append(e_cur)
        i = arg
    if d == 0:
        raise OracleError(3, "decompose: start column is numerically zero, no basis built")
    out = OracleModel(Y[:, :d].copy(order="F"), T[:d].copy(), sel, hist, d)
    out.col_sq = col_sq
    return out


def column_sq(x, nthreads: int = 1) -> np.ndarray:
    """||x_j||^2 per column in the oracle's dot8 order (workspace.cpp:22)."""
    xa = np.asfortranarray(np.asarray(x, dtype=np.float64))
    m, n = xa.shape
    out = np.zeros(n)
    f, z = C.c_int(), C.c_int()
    lib().orc_column_pass(_p(xa), m, n, xa.strides[1] // 8 if n > 1 else m, int(nthreads),
                          _p(out), C.byref(f), C.byref(z))
    return out


def mgs_project(v, basis, breakdown_tol: float, reorthogonalize: bool = False):
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
    m = v.shape[0]
    if basis is None or np.asarray(basis).size == 0:
        B, k = np.zeros((m, 1), order="F"), 0
    else:
        B = np.asfortranarray(np.asarray(basis, dtype=np.float64))
        k = B.shape[1]
    xi = np.zeros(m)
    nrm = C.c_double()
    ok = lib().orc_mgs_project(_p(v), m, _p(B), k, m, float(breakdown_tol),
                               1 if reorthogonalize else 0, _p(xi), C.byref(nrm))
    if not ok:
        return None
    return xi, nrm.value


class Workspace:
    """ErrorWorkspace, identity or diagonal weight (workspace.cpp:9-125)."""

    def __init__(self, x, diag=None):
        self.x = np.asfortranarray(np.asarray(x, dtype=np.float64))
        self.m, self.n = self.x.shape
        self.h = None
        if diag is None:
            self.h = lib().orc_ws_init(_p(self.x), self.m, self.n, self.m)
        else:
            self.diag = np.ascontiguousarray(np.asarray(diag, dtype=np.float64).reshape(-1))
            self.h = lib().orc_ws_init_diag(_p(self.x), self.m, self.n, self.m, _p(self.diag),
                                            self.diag.size)
            if not self.h:
                raise OracleError(ORC_INCOMPATIBLE_WEIGHT, lib().orc_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_ws_free(self.h)
            self.h = None

    @property
    def d(self):
        return lib().orc_ws_d(self.h)

    def extend(self, xi):
        xi = np.ascontiguousarray(np.asarray(xi, dtype=np.float64))
        lib().orc_ws_extend(self.h, _p(xi))

    def col_sq(self):
        out = np.zeros(self.n)
        lib().orc_ws_col_sq(self.h, _p(out))
        return out

    def residual(self):
        out = np.zeros(self.n)
        lib().orc_ws_residual(self.h, _p(out))
        return out

    def yax_row(self, k):
        out = np.zeros(self.n)
        lib().orc_ws_yax_row(self.h, int(k), _p(out))
        return out

    def error_sq(self, j, c):
        c = np.ascontiguousarray(np.asarray(c, dtype=np.float64).reshape(-1))
        out = C.c_double()
        rc = lib().orc_ws_error_sq(self.h, int(j), _p(c) if c.size else None, c.shape[0],
                                   C.byref(out))
        if rc != ORC_OK:
            raise OracleError(rc, lib().orc_last_error().decode())
        return out.value

    def scan_T(self, T):
        """residual_scan(ws, T) for any weight (T is d x n)."""
        Ta = np.ascontiguousarray(np.asarray(T, dtype=np.float64))
        e = C.c_double()
        j = C.c_int64()
        lib().orc_ws_scan_T(self.h, _p(Ta), C.byref(e), C.byref(j))
        return e.value, j.value

    def yay(self):
        d = self.d
        out = np.zeros((d, d))
        lib().orc_ws_yay(self.h, _p(out))
        return out

    def scan(self):
        e = C.c_double()
        j = C.c_int64()
        lib().orc_ws_scan(self.h, C.byref(e), C.byref(j))
        return e.value, j.value


def project(Y, v):
    """rbd::project (decompose.cpp:113-117): c = Y'v for one vector, the
    reference's per-vector call (Y re-read per vector)."""
    Ya = np.asfortranarray(np.asarray(Y, dtype=np.float64))
    va = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))
    m, d = Ya.shape
    c = np.zeros(d)
    lib().orc_project(_p(Ya), m, d, _p(va), _p(c))
    return c


def project_batch(Y, Xn, nthreads: int = 1):
    Ya = np.asfortranarray(np.asarray(Y, dtype=np.float64))
    Xa = np.asfortranarray(np.asarray(Xn, dtype=np.float64))
    m, d = Ya.shape
    N = Xa.shape[1]
    Tn = np.zeros((d, N), order="F")
    err = np.zeros(N)
    lib().orc_project_batch(_p(Ya), m, d, _p(Xa), N, m, int(nthreads), _p(Tn), _p(err))
    return Tn, err


def random_positive(n, seed):
    """testutil::random_positive (helpers.hpp:28-34), bit-identical draws."""
    out = np.zeros(n)
    lib().orc_random_positive(int(n), int(seed) & 0xFFFFFFFFFFFFFFFF, _p(out))
    return out


def random_matrix(m, n, seed):
    """testutil::random_matrix (helpers.hpp:14-21), bit-identical draws."""
    out = np.zeros((m, n), order="F")
    lib().orc_random_matrix(m, n, int(seed), _p(out))
    return out


def random_low_rank(m, n, r, seed):
    out = np.zeros((m, n), order="F")
    lib().orc_random_low_rank(m, n, r, int(seed), _p(out))
    return out


GRID_FUNCS = {"rank1": 0, "rank2": 1, "rank3": 2, "composite": 3}


def gen_grid_matrix(name: str, n_points: int = 101):
    out = np.zeros((n_points, n_points), order="F")
    rc = lib().orc_gen_grid_matrix(GRID_FUNCS[name], n_points, _p(out))
    if rc != ORC_OK:
        raise OracleError(rc, lib().orc_last_error().decode())
    return out


def acceptance3_count() -> int:
    return int(lib().orc_acceptance3_count())


def seeded_start(seed: int, n: int) -> int:
    return int(lib().orc_seeded_start(int(seed) & 0xFFFFFFFFFFFFFFFF, int(n)))


# ---- RBD1 model container, restated (proj/src/io.cpp:527-622, io.hpp:51-64) ----

def model_bytes(Y, T, eps_r, history, tag=0, diag=None) -> bytes:
    """write_model's byte stream (io.cpp:533-570): "RBD1", u64 m/n/d, u8 tag,
    Y column-major, T row-major, eps_R, history, (tag 1) diag; little-endian."""
    import struct
    Y = np.asarray(Y, dtype=np.float64)
    T = np.asarray(T, dtype=np.float64)
    m, d = Y.shape
    n = T.shape[1]
    assert T.shape[0] == d, "write_model: inconsistent model shapes"     # io.cpp:537-538
    out = [b"RBD1", struct.pack("<QQQB", m, n, d, tag),                    # :556-560
           np.asarray(Y, dtype="<f8").tobytes(order="F"),                   # :561-562
           np.asarray(T, dtype="<f8").tobytes(order="C"),                   # :563-564
           struct.pack("<d", float(eps_r)),                                 # :565
           np.asarray(history, dtype="<f8").tobytes()]                      # :566-567
    if tag == 1:
        out.append(np.asarray(diag, dtype="<f8").tobytes())                # :568-569
    return b"".join(out)


def parse_model(data: bytes):
    """read_model (io.cpp:574-622): returns (Y, T, eps_r, history, tag, diag) or
    raises ValueError with the reference's ParseError text."""
    import struct
    if len(data) < 29 or data[:4] != b"RBD1":
        raise ValueError("not a model file (bad magic)")                    # :580-581
    m, n, d, tag = struct.unpack_from("<QQQB", data, 4)
    if m < 1 or n < 1 or d < 1 or d > n:
        raise ValueError("implausible model dimensions")                    # :587-588
    if tag > 2:
        raise ValueError("unknown weight tag")                              # :590
    expected = 29 + 8 * (m * d + d * n + 1 + d) + (8 * m if tag == 1 else 0)
    if len(data) != expected:
        raise ValueError("model file size does not match header")           # :592-596
    f = np.frombuffer(data, dtype="<f8", offset=29)
    Y = f[: m * d].reshape((m, d), order="F")
    T = f[m * d: m * d + d * n].reshape((d, n))
    eps_r = float(f[m * d + d * n])
    hist = f[m * d + d * n + 1: m * d + d * n + 1 + d]
    diag = f[m * d + d * n + 1 + d:] if tag == 1 else None
    return Y, T, eps_r, hist, tag, diag


# ---- Classifier (classify.cpp:11-48), restated ----

def predict_batch(Y, T, Qm, nthreads: int = 1):
    """Best training column and squared distance per query (classify.cpp:22-34)."""
    Ya = np.asfortranarray(np.asarray(Y, dtype=np.float64))
    Ta = np.ascontiguousarray(np.asarray(T, dtype=np.float64))
    Qa = np.asfortranarray(np.asarray(Qm, dtype=np.float64))
    if Qa.ndim == 1:
        Qa = Qa.reshape(-1, 1, order="F")
    m, d = Ya.shape
    n_tr = Ta.shape[1]
    nq = Qa.shape[1]
    best = np.zeros(nq, dtype=np.int64)
    dist = np.zeros(nq)
    lib().orc_predict_batch(_p(Ya), m, d, _p(Ta), n_tr, _p(Qa), nq, int(nthreads), _p(best),
                            _p(dist))
    return best, dist


def gen_labeled_blobs(n_classes, per_class, dim, spread, seed):
    """datasets.cpp:67-97 (samples dim x n, integer labels), bit-identical draws."""
    n = n_classes * per_class
    samples = np.zeros((dim, n), order="F")
    labels = np.zeros(n, dtype=np.int32)
    rc = lib().orc_gen_labeled_blobs(int(n_classes), int(per_class), int(dim), float(spread),
                                     int(seed) & 0xFFFFFFFFFFFFFFFF, _p(samples), _p(labels))
    if rc != ORC_OK:
        raise OracleError(rc, lib().orc_last_error().decode())
    return samples, labels
