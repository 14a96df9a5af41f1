"""ctypes binding of the C ABI declared in include/rbd_cuda.h.

The product path has no CPU fallback: if ``librbd_b200.so`` is missing or
fails to load, importing the compute API raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from ._build import LIB

# ---- status codes (include/rbd_cuda.h) ----
RBD_OK = 0
RBD_ERR_INVALID_ARGUMENT = 1
RBD_ERR_INCOMPATIBLE_WEIGHT = 2
RBD_ERR_DEGENERATE_INPUT = 3
RBD_ERR_INDEX_OUT_OF_RANGE = 4
RBD_ERR_DIMENSION_MISMATCH = 5
RBD_ERR_NOT_POSITIVE = 6
RBD_ERR_NO_CONVERGENCE = 7
RBD_ERR_UNSUPPORTED_FORMAT = 8
RBD_ERR_IO = 9
RBD_ERR_PARSE = 10
RBD_ERR_CUDA = 100
RBD_ERR_NCCL = 101
RBD_ERR_OUT_OF_MEMORY = 102


class RbdError(RuntimeError):
    """Base error (the reference's rbd::Error, errors.hpp:9-12; pybind RbdError)."""


class InvalidArgument(RbdError):
    pass


class IncompatibleWeight(RbdError):
    pass


class DegenerateInput(RbdError):
    pass


class IndexOutOfRange(RbdError):
    pass


class DimensionMismatch(RbdError):
    pass


class NotPositive(RbdError):
    pass


class NoConvergence(RbdError):
    pass


class UnsupportedFormat(RbdError):
    pass


class IoError(RbdError):
    pass


class ParseError(RbdError):
    """errors.hpp:64-77; the message is "path:line: what"."""


class CudaError(RbdError):
    pass


_ERRORS = {
    RBD_ERR_INVALID_ARGUMENT: InvalidArgument,
    RBD_ERR_INCOMPATIBLE_WEIGHT: IncompatibleWeight,
    RBD_ERR_DEGENERATE_INPUT: DegenerateInput,
    RBD_ERR_INDEX_OUT_OF_RANGE: IndexOutOfRange,
    RBD_ERR_DIMENSION_MISMATCH: DimensionMismatch,
    RBD_ERR_NOT_POSITIVE: NotPositive,
    RBD_ERR_NO_CONVERGENCE: NoConvergence,
    RBD_ERR_UNSUPPORTED_FORMAT: UnsupportedFormat,
    RBD_ERR_IO: IoError,
    RBD_ERR_PARSE: ParseError,
}


class Config(C.Structure):
    """rbd_config_t — mirrors rbd::RbdConfig (decompose.hpp:25-36)."""
    _fields_ = [
        ("d_max", C.c_int64),
        ("eps_R", C.c_double),
        ("start_kind", C.c_int32),
        ("reorthogonalize", C.c_int32),
        ("start_column", C.c_int64),
        ("start_seed", C.c_uint64),
        ("breakdown_tol", C.c_double),
        ("weight_kind", C.c_int32),
        ("weight_dim", C.c_int64),
    ]


class Result(C.Structure):
    _fields_ = [
        ("d", C.c_int64),
        ("breakdown", C.c_int32),
        ("reserved", C.c_int32),
        ("breakdown_tol", C.c_double),
        ("max_col_norm", C.c_double),
        ("init_ms", C.c_double),
        ("loop_ms", C.c_double),
        ("launches", C.c_int64),
    ]


_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double
_DP = C.POINTER(C.c_double)
_I64P = C.POINTER(C.c_int64)

_SIGS = {
    "rbd_last_error": (C.c_char_p, []),
    "rbd_abi_version": (C.c_int, []),
    "rbd_config_default": (None, [C.POINTER(Config)]),
    "rbd_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "rbd_ctx_destroy": (C.c_int, [_P]),
    "rbd_ctx_set_stream": (C.c_int, [_P, _P]),
    "rbd_ctx_launch_count": (C.c_int64, [_P]),
    "rbd_set_forced_selection": (C.c_int, [_P, _P, C.c_int64]),
    "rbd_ctx_synchronize": (C.c_int, [_P]),
    "rbd_ctx_stream": (_P, [_P]),
    "rbd_decompose_device": (C.c_int, [_P, _P, _I64, _I64, _I64, C.POINTER(Config), _P, _P, _P, _P,
                                       C.POINTER(Result)]),
    "rbd_decompose_host": (C.c_int, [_P, _P, _I64, _I64, _I64, C.POINTER(Config), _P, _P, _P, _P,
                                     C.POINTER(Result)]),
    "rbd_decompose_host_many": (C.c_int, [_P, _I64, _P, _I64, _I64, _I64, C.POINTER(Config), _P, _P,
                                          _P, _P, _P]),
    "rbd_decompose_host_many_f32": (C.c_int, [_P, _I64, _P, _I64, _I64, _I64, C.POINTER(Config), _P,
                                              _P, _P, _P, _P]),
    "rbd_decompose_host_f32": (C.c_int, [_P, _P, _I64, _I64, _I64, C.POINTER(Config), _P, _P, _P, _P,
                                     C.POINTER(Result)]),
    "rbd_decompose_device_f32": (C.c_int, [_P, _P, _I64, _I64, _I64, C.POINTER(Config), _P, _P, _P, _P,
                                       C.POINTER(Result)]),
    "rbd_classify_batch": (C.c_int, [_P, _P, _I64, _I64, _I64, _P, _I64, _P, _I64, _I64, _P, _P]),
    "rbd_classify_host": (C.c_int, [_P, _P, _I64, _I64, _P, _I64, _P, _I64, _P, _P]),
    "rbd_nearest_columns": (C.c_int, [_P, _P, _I64, _I64, _I64, _P, _I64, _P, _P]),
    "rbd_compress_device": (C.c_int, [_P, _P, _I64, _I64, _I64, _P, _I64, _I64, _P, _I64]),
    "rbd_ws_init_diag": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, _P, _I64, C.POINTER(_P)]),
    "rbd_ws_init_diag_host": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, _P, _I64, C.POINTER(_P)]),
    "rbd_ws_scan_T": (C.c_int, [_P, _P, C.POINTER(C.c_double), C.POINTER(_I64)]),
    "rbd_ws_scan_T_host": (C.c_int, [_P, _P, C.POINTER(C.c_double), C.POINTER(_I64)]),
    "rbd_ws_read_yay": (C.c_int, [_P, _P]),
    "rbd_model_write": (C.c_int, [_P, C.c_char_p, _I64, _I64, _I64, _P, _I64, _P, C.c_double, _P,
                                  C.c_int, _P]),
    "rbd_model_read_header": (C.c_int, [C.c_char_p, C.POINTER(_I64), C.POINTER(_I64),
                                        C.POINTER(_I64), C.POINTER(C.c_int)]),
    "rbd_model_read": (C.c_int, [_P, C.c_char_p, _P, _I64, _P, C.POINTER(C.c_double), _P, _P]),
    "rbd_decompose_diag_device": (C.c_int, [_P, _P, _I64, _I64, _I64, C.POINTER(Config), _P, _I64,
                                            _P, _P, _P, _P, C.POINTER(Result)]),
    "rbd_decompose_diag_host": (C.c_int, [_P, _P, _I64, _I64, _I64, C.POINTER(Config), _P, _I64,
                                          _P, _P, _P, _P, C.POINTER(Result)]),
    "rbd_mgs_project": (C.c_int, [_P, _P, _I64, _P, _I64, _I64, _D, C.c_int, _P, _DP,
                                  C.POINTER(C.c_int)]),
    "rbd_ws_init": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, C.POINTER(_P)]),
    "rbd_ws_destroy": (C.c_int, [_P]),
    "rbd_ws_extend": (C.c_int, [_P, _P]),
    "rbd_ws_scan": (C.c_int, [_P, _DP, _I64P]),
    "rbd_ws_error_sq": (C.c_int, [_P, _I64, _P, _I64, _DP]),
    "rbd_ws_d": (C.c_int64, [_P]),
    "rbd_ws_read": (C.c_int, [_P, _P, _P, _P]),
    "rbd_project_batch": (C.c_int, [_P, _P, _I64, _I64, _I64, _P, _I64, _I64, _P, _P]),
    "rbd_reconstruct": (C.c_int, [_P, _P, _I64, _I64, _I64, _P, _P]),
    "rbd_project_batch_f32": (C.c_int, [_P, _P, _I64, _I64, _I64, _P, _I64, _I64, _P, _P]),
    "rbd_project_host": (C.c_int, [_P, _P, _I64, _I64, _P, _I64, _P, _P]),
    "rbd_reconstruct_host": (C.c_int, [_P, _P, _I64, _I64, _P, _P]),
    "rbd_time_sweep": (C.c_int, [_P, _P, _I64, _I64, _I64, _P, C.c_int, _DP]),
    "rbd_comm_unique_id": (C.c_int, [C.c_char_p]),
    "rbd_shard_pick": (C.c_int, [_P, C.c_int, C.POINTER(C.c_double), C.POINTER(_I64),
                                 C.POINTER(C.c_int)]),
    "rbd_ctx_init_comm": (C.c_int, [_P, C.c_int, C.c_int, C.c_char_p]),
    "rbd_decompose_sharded": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, _I64, C.POINTER(Config),
                                        _P, _P, _P, _P, C.POINTER(Result)]),
    "rbd_mgs_project_host": (C.c_int, [_P, _P, _I64, _P, _I64, _I64, _D, C.c_int, _P, _DP,
                                       C.POINTER(C.c_int)]),
    "rbd_ws_init_host": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, C.POINTER(_P)]),
    "rbd_ws_extend_host": (C.c_int, [_P, _P]),
    "rbd_reconstruct_batch": (C.c_int, [_P, _P, _I64, _I64, _I64, _P, _I64, _P]),
    "rbd_compress_host": (C.c_int, [_P, _P, _I64, _I64, _P, _I64, _P]),
    "rbd_decompose_sharded_virtual": (C.c_int, [_P, C.c_int, _P, _P, _I64, _I64, C.POINTER(Config),
                                                _P, _P, _P, _P, C.POINTER(Result)]),
    "rbd_model_create": (C.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P, C.c_int, _P, C.c_double,
                                   C.POINTER(_P)]),
    "rbd_model_load": (C.c_int, [_P, C.c_char_p, C.POINTER(_P)]),
    "rbd_model_free": (C.c_int, [_P]),
    "rbd_model_info": (C.c_int, [_P, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64),
                                 C.POINTER(_P), C.POINTER(_P), C.POINTER(C.c_double),
                                 C.POINTER(C.c_int)]),
    "rbd_model_read_vectors": (C.c_int, [_P, _P, _P]),
    "rbd_project_model": (C.c_int, [_P, _P, _P, _I64, _I64, _P, _P]),
    "rbd_reconstruct_model": (C.c_int, [_P, _P, _P, _I64, _P]),
    "rbd_project_host_many": (C.c_int, [_P, _P, _I64, _P, _I64, _I64, _P, _P]),
    "rbd_project_host_many_f32": (C.c_int, [_P, _P, _I64, _P, _I64, _I64, _P, _P]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB):
    """Load librbd_b200.so (raises if it is absent: no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int) -> None:
    if status == RBD_OK:
        return
    msg = (load_library().rbd_last_error() or b"").decode()
    raise _ERRORS.get(status, CudaError if status >= 100 else RbdError)(msg)


def default_config(d_max: int = 1) -> Config:
    cfg = Config()
    load_library().rbd_config_default(C.byref(cfg))
    cfg.d_max = d_max
    return cfg


class Context:
    """One rbd_ctx (device, stream, scratch, captured graphs)."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = _P()
        check(lib.rbd_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device
        self._lib = lib

    def close(self):
        if self.handle:
            self._lib.rbd_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self._lib.rbd_ctx_launch_count(self.handle))

    @property
    def stream(self) -> int:
        return int(self._lib.rbd_ctx_stream(self.handle) or 0)

    def synchronize(self):
        check(self._lib.rbd_ctx_synchronize(self.handle))

    def force_selection(self, selected=None):
        """Parity-protocol instrumentation: later decompose calls on
        this context follow `selected` instead of the greedy argmax (None clears)."""
        import numpy as np
        arr = np.ascontiguousarray(np.asarray([] if selected is None else selected,
                                              dtype=np.int64).reshape(-1))
        check(self._lib.rbd_set_forced_selection(
            self.handle, arr.ctypes.data_as(C.c_void_p) if arr.size else None, arr.size))


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]
