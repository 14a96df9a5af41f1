"""Python mirror of the reference's RBD API (proj/python/bindings.cpp:41-178,
proj/include/rbd/decompose.hpp:61-77, workspace.hpp:34-54), executed on B200
through the C ABI (include/rbd_cuda.h).

Host arrays (numpy) go through the reference-facing host entry points
(upload -> CUDA loop -> download inside the call); torch CUDA tensors go
through the device-resident entry points. There is no CPU compute path.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import _lib
from ._lib import (Config, Context, DimensionMismatch, InvalidArgument, Result, check,
                   default_config, default_context, load_library)

try:  # torch is plumbing (device memory / streams); optional for host calls
    import torch
except Exception:  # pragma: no cover
    torch = None


def _is_torch_cuda(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _col_major_np(x) -> np.ndarray:
    return np.asfortranarray(np.asarray(x, dtype=np.float64))


def _col_major_torch(x, dtype=None):
    dtype = dtype or torch.float64
    if x.dtype != dtype:
        x = x.to(dtype)
    if x.dim() != 2:
        raise InvalidArgument("decompose: X must be a 2-D matrix")
    m = x.shape[0]
    if x.stride(0) == 1 and x.stride(1) >= max(m, 1):
        return x, x.stride(1)
    xc = x.t().contiguous().t()
    return xc, m


def output_buffers(m: int, n: int, d_max: int, count: int = 1):
    """Page-locked (Y, T) output pairs for decompose_many(out=...): Y m x cap
    column-major, T cap x n row-major, cap = min(d_max, n)."""
    cap = max(1, min(int(d_max), n)) if n > 0 else 1
    return [_host_outputs(m, n, cap) for _ in range(count)]


def _host_outputs(m: int, n: int, cap: int):
    """Y (m x cap, column-major) and T (cap x n) host buffers; page-locked when
    torch is available so the device-to-host copies run at full PCIe rate."""
    if torch is not None and torch.cuda.is_available() and m * cap + cap * n >= (1 << 20):
        Yt = torch.empty((cap, max(m, 1)), dtype=torch.float64, pin_memory=True)
        Tt = torch.empty((cap, max(n, 1)), dtype=torch.float64, pin_memory=True)
        return Yt.numpy().T, Tt.numpy()
    return (np.zeros((m, cap), dtype=np.float64, order="F"),
            np.zeros((cap, n), dtype=np.float64))


F32_MAX_D = 4096   # the persistent loop's limit (kFMaxCoef, csrc/rbd_device.cuh)


def _auto_storage(x, d_max, identity: bool) -> str:
    dt = getattr(x, "dtype", None)
    is32 = dt in ((torch.float32,) if torch is not None else ()) + (np.float32,)
    if is32 and identity and int(d_max) <= F32_MAX_D and os.environ.get("RBD_PATH", "") != "graph":
        return "f32"
    return "f64"


def make_config(d_max: int, eps_r: float = 0.0, start_column: int = 0,
                reorthogonalize: bool = False, breakdown_tol: float = -1.0,
                start_seed: Optional[int] = None, diag=None, sparse=None) -> Config:
    """config_from_args (bindings.cpp:27-37) + RbdConfig defaults (decompose.hpp:25-36)."""
    if diag is not None and sparse is not None:
        raise InvalidArgument("pass at most one of diag and sparse")
    cfg = default_config(int(d_max))
    cfg.eps_R = float(eps_r)
    cfg.reorthogonalize = 1 if reorthogonalize else 0
    cfg.breakdown_tol = float(breakdown_tol)
    if start_seed is not None:
        cfg.start_kind = 1
        cfg.start_seed = int(start_seed) & 0xFFFFFFFFFFFFFFFF
    else:
        cfg.start_kind = 0
        cfg.start_column = int(start_column)
    if diag is not None:
        cfg.weight_kind = 1
        cfg.weight_dim = int(diag.shape[0]) if hasattr(diag, "shape") else len(diag)
    elif sparse is not None:
        cfg.weight_kind = 2
        cfg.weight_dim = int(sparse.shape[0])
    return cfg


class Model:
    """RbdModel (decompose.hpp:39-46): X ~= Y T with Y'Y = I.

    ``Y`` is m x d, ``T`` is d x n (numpy for host calls, torch CUDA tensors for
    device calls); ``selected`` and ``residual_history`` are Python lists.
    """

    def __init__(self, Y, T, d, selected, residual_history, result: Result, ctx: Context,
                 weight_kind: int = 0, diag=None):
        self._Y = Y
        self._T = T
        self.d = int(d)
        self.selected = list(int(s) for s in selected)
        self.residual_history = list(float(h) for h in residual_history)
        self.result = result
        self._ctx = ctx
        # RbdModel::weight (decompose.hpp:45): 0 identity, 1 diagonal (values in
        # `diag`, host numpy), 2 sparse SPD held externally (loaded models only)
        self.weight_kind = int(weight_kind)
        self.diag = None if diag is None else np.ascontiguousarray(
            diag.detach().cpu().numpy() if hasattr(diag, "detach") else np.asarray(diag),
            dtype=np.float64).reshape(-1)
        self._resident = None

    def resident(self) -> "ResidentModel":
        """The device-resident copy of a host model (rbd_model_t), made on first
        use and reused by project / reconstruct: no Y upload per call."""
        if self._resident is None:
            self._resident = ResidentModel.from_model(self, ctx=self._ctx)
        return self._resident

    @property
    def Y(self):
        return self._Y[:, : self.d]

    @property
    def T(self):
        return self._T[: self.d]

    @property
    def on_device(self) -> bool:
        return _is_torch_cuda(self._Y)

    def project(self, v):
        """Reduced coordinates c = Y'v (decompose.cpp:113-117)."""
        return project(self, v)

    def reconstruct(self, c):
        """Y c (decompose.cpp:119-123)."""
        return reconstruct(self, c)

    def save(self, path, eps_r: float = 0.0):
        """Model.save (bindings.cpp:63-67) -> write_model (io.cpp:533-570): the RBD1
        container, written atomically; device-resident Y/T stream from HBM."""
        return save(self, path, eps_r)

    def compress(self):
        """compress_matrix: Y T (decompose.cpp:125) on the FP64 tensor cores
        (rbd_compress_device / rbd_compress_host)."""
        lib = load_library()
        Y, T = self.Y, self.T
        m, d = Y.shape
        n = T.shape[1]
        if self.on_device:
            Yc = Y if Y.stride(0) == 1 else Y.t().contiguous().t()
            Tc = T.contiguous()
            V = torch.empty((n, m), dtype=torch.float64, device=Y.device).t()
            ctx = self._ctx or default_context(Y.device.index or 0)
            torch.cuda.current_stream(Y.device).synchronize()
            check(lib.rbd_compress_device(ctx.handle, C.c_void_p(Yc.data_ptr()), m, d,
                                          Yc.stride(1) if d > 1 else m,
                                          C.c_void_p(Tc.data_ptr()), n, n,
                                          C.c_void_p(V.data_ptr()), m))
            ctx.synchronize()
            return V
        ctx = self._ctx or default_context(0)
        Yh = np.asfortranarray(Y)
        Ch = np.asfortranarray(T)        # d x n column-major coefficients
        V = np.zeros((m, n), order="F")
        check(lib.rbd_compress_host(ctx.handle, _dp(Yh), m, d, _dp(Ch), n, _dp(V)))
        return V


def decompose(x, d_max: int, eps_r: float = 0.0, diag=None, sparse=None, start_column: int = 0,
              reorthogonalize: bool = False, breakdown_tol: float = -1.0,
              start_seed: Optional[int] = None, ctx: Optional[Context] = None,
              forced_selection=None, storage: Optional[str] = None) -> Model:
    """rbd.decompose (bindings.cpp:69-78) -> rbd::decompose (decompose.cpp:53-111).

    numpy input: end-to-end host entry (rbd_decompose_host).
    torch CUDA input: device-resident entry (rbd_decompose_device).
    storage: "f64" or "f32". Default: "f32" for float32 input when the fp32
    mode applies (identity weight, persistent loop: d_max <= 4096 and
    RBD_PATH unset), else "f64" — float32 input is widened exactly, as the
    reference's binding converts it to a double Matrix.
    "f32" keeps X in fp32 on the device (rbd_decompose_*_f32: half the bytes
    per sweep, fp64 arithmetic on the fp32 values; identity weight only).
    forced_selection: parity-test instrumentation; follow this
    column sequence instead of the greedy argmax (persistent loop only).
    """
    if forced_selection is not None:
        ctx = ctx or default_context((x.device.index or 0) if _is_torch_cuda(x) else 0)
        ctx.force_selection(forced_selection)
        try:
            return decompose(x, d_max, eps_r, diag, sparse, start_column, reorthogonalize,
                             breakdown_tol, start_seed, ctx, storage=storage)
        finally:
            ctx.force_selection(None)
    if storage is None:
        storage = _auto_storage(x, d_max, diag is None and sparse is None)
    if storage not in ("f32", "f64"):
        raise InvalidArgument("decompose: storage must be 'f32' or 'f64'")
    f32 = storage == "f32"
    if f32 and (diag is not None or sparse is not None):
        raise InvalidArgument("decompose: fp32 storage mode supports the identity weight only")
    cfg = make_config(d_max, eps_r, start_column, reorthogonalize, breakdown_tol, start_seed,
                      diag, sparse)
    lib = load_library()
    res = Result()
    if _is_torch_cuda(x):
        dev = x.device.index or 0
        ctx = ctx or default_context(dev)
        xc, ldx = _col_major_torch(x, torch.float32 if f32 else torch.float64)
        m, n = xc.shape
        cap = max(1, min(int(d_max), n)) if n > 0 else 1
        Y = torch.empty((cap, max(m, 1)), dtype=torch.float64, device=x.device).t()
        T = torch.empty((cap, max(n, 1)), dtype=torch.float64, device=x.device)
        sel = np.zeros(cap, dtype=np.int64)
        hist = np.zeros(cap, dtype=np.float64)
        torch.cuda.current_stream(x.device).synchronize()
        if diag is not None:   # WeightSpec::diagonal
            dg = torch.as_tensor(diag, dtype=torch.float64, device=x.device).reshape(-1).contiguous()
            torch.cuda.current_stream(x.device).synchronize()
            check(lib.rbd_decompose_diag_device(
                ctx.handle, C.c_void_p(xc.data_ptr()), m, n, ldx, C.byref(cfg),
                C.c_void_p(dg.data_ptr()) if dg.numel() else None, dg.numel(),
                C.c_void_p(Y.data_ptr()), C.c_void_p(T.data_ptr()), _dp(sel), _dp(hist),
                C.byref(res)))
        else:
            fn = lib.rbd_decompose_device_f32 if f32 else lib.rbd_decompose_device
            check(fn(ctx.handle, C.c_void_p(xc.data_ptr()), m, n, ldx, C.byref(cfg),
                     C.c_void_p(Y.data_ptr()), C.c_void_p(T.data_ptr()), _dp(sel), _dp(hist),
                     C.byref(res)))
        d = res.d
        return Model(Y, T, d, sel[:d], hist[:d], res, ctx, 1 if diag is not None else 0, diag)
    ctx = ctx or default_context(0)
    xa = np.asfortranarray(np.asarray(x, dtype=np.float32)) if f32 else _col_major_np(x)
    if xa.ndim != 2:
        raise InvalidArgument("decompose: X must be a 2-D matrix")
    m, n = xa.shape
    cap = max(1, min(int(d_max), n)) if n > 0 else 1
    Y, T = _host_outputs(m, n, cap)
    sel = np.zeros(cap, dtype=np.int64)
    hist = np.zeros(cap, dtype=np.float64)
    if diag is not None:   # WeightSpec::diagonal
        dg = np.ascontiguousarray(np.asarray(diag, dtype=np.float64).reshape(-1))
        check(lib.rbd_decompose_diag_host(ctx.handle, _dp(xa), m, n, max(m, 1), C.byref(cfg),
                                          _dp(dg) if dg.size else None, dg.size, _dp(Y), _dp(T),
                                          _dp(sel), _dp(hist), C.byref(res)))
    else:
        fn = lib.rbd_decompose_host_f32 if f32 else lib.rbd_decompose_host
        check(fn(ctx.handle, _dp(xa), m, n, max(m, 1), C.byref(cfg), _dp(Y), _dp(T), _dp(sel),
                 _dp(hist), C.byref(res)))
    d = res.d
    return Model(Y, T, d, sel[:d], hist[:d], res, ctx, 1 if diag is not None else 0, diag)


def decompose_many(xs, d_max: int, eps_r: float = 0.0, start_column: int = 0,
                   reorthogonalize: bool = False, breakdown_tol: float = -1.0,
                   start_seed: Optional[int] = None, ctx: Optional[Context] = None,
                   storage: Optional[str] = None, out=None):
    """rbd::decompose over a sequence of host matrices of one shape
    (rbd_decompose_host_many): the upload of matrix i+1 overlaps the greedy
    loop of matrix i. Returns one Model per matrix. Page-locked inputs (e.g.
    ``torch.empty(..., pin_memory=True).numpy()``) are needed for the overlap.
    ``out`` may pass one (Y, T) pair of host buffers per matrix (Y m x cap
    column-major, T cap x n row-major, cap = min(d_max, n); see
    ``output_buffers``) that the models then view — e.g. page-locked buffers
    reused across calls."""
    xs = list(xs)
    if not xs:
        return []
    if storage is None:
        storage = "f32" if all(_auto_storage(x, d_max, True) == "f32" for x in xs) else "f64"
    if storage not in ("f32", "f64"):
        raise InvalidArgument("decompose: storage must be 'f32' or 'f64'")
    f32 = storage == "f32"
    dt = np.float32 if f32 else np.float64
    arrs = []
    for x in xs:
        a = x if (isinstance(x, np.ndarray) and x.dtype == dt and x.flags["F_CONTIGUOUS"]) \
            else np.asfortranarray(np.asarray(x, dtype=dt))
        if a.ndim != 2 or a.shape != np.shape(arrs[0] if arrs else a):
            raise InvalidArgument("decompose_many: matrices must be 2-D and of one shape")
        arrs.append(a)
    m, n = arrs[0].shape
    cfg = make_config(d_max, eps_r, start_column, reorthogonalize, breakdown_tol, start_seed)
    lib = load_library()
    ctx = ctx or default_context(0)
    cap = max(1, min(int(d_max), n)) if n > 0 else 1
    cnt = len(arrs)
    if out is not None:
        outs = list(out)
        if len(outs) != cnt or any(
                np.shape(o[0]) != (m, cap) or np.shape(o[1]) != (cap, n)
                or o[0].dtype != np.float64 or o[1].dtype != np.float64
                or not o[0].flags["F_CONTIGUOUS"] or not o[1].flags["C_CONTIGUOUS"] for o in outs):
            raise InvalidArgument("decompose_many: out needs one (Y m x cap F-order, "
                                  "T cap x n C-order) float64 pair per matrix")
    else:
        outs = [_host_outputs(m, n, cap) for _ in range(cnt)]
    sels = [np.zeros(cap, dtype=np.int64) for _ in range(cnt)]
    hists = [np.zeros(cap, dtype=np.float64) for _ in range(cnt)]
    res = (Result * cnt)()
    P = C.c_void_p * cnt
    xp = P(*[a.ctypes.data for a in arrs])
    yp = P(*[o[0].ctypes.data for o in outs])
    tp = P(*[o[1].ctypes.data for o in outs])
    sp = P(*[v.ctypes.data for v in sels])
    hp = P(*[v.ctypes.data for v in hists])
    fn = lib.rbd_decompose_host_many_f32 if f32 else lib.rbd_decompose_host_many
    check(fn(ctx.handle, cnt, xp, m, n, max(m, 1), C.byref(cfg), yp, tp, sp, hp, res))
    return [Model(outs[i][0], outs[i][1], res[i].d, sels[i][:res[i].d], hists[i][:res[i].d],
                  res[i], ctx) for i in range(cnt)]


def _ptr(a):
    return C.c_void_p(a.data_ptr()) if hasattr(a, "data_ptr") else _dp(a)


def save(model: Model, path, eps_r: float = 0.0):
    """write_model (io.cpp:533-570) through rbd_model_write."""
    lib = load_library()
    Y, T = model.Y, model.T
    if _is_torch_cuda(Y):
        Yc = Y if Y.stride(0) == 1 else Y.t().contiguous().t()
        Tc = T.contiguous()
        ldy = Yc.stride(1) if Yc.dim() == 2 and Yc.shape[1] > 1 else Yc.shape[0]
        torch.cuda.current_stream(Y.device).synchronize()
    else:
        Yc = np.asfortranarray(Y)
        Tc = np.ascontiguousarray(T)
        ldy = Yc.shape[0]
    m, d = Yc.shape
    n = Tc.shape[1]
    hist = np.ascontiguousarray(np.asarray(model.residual_history, dtype=np.float64))
    if d != model.d or Tc.shape[0] != model.d or hist.shape[0] != model.d:   # io.cpp:537-538
        raise DimensionMismatch("write_model: inconsistent model shapes")
    if model.weight_kind == 1 and (model.diag is None or model.diag.shape[0] != m):
        raise DimensionMismatch("write_model: diagonal weight length != m")
    diag = model.diag if model.weight_kind == 1 else None
    ctx = model._ctx
    check(lib.rbd_model_write(ctx.handle if ctx is not None else None, os.fsencode(str(path)), m,
                              n, d, _ptr(Yc), ldy, _ptr(Tc), float(eps_r), _dp(hist),
                              model.weight_kind, _dp(diag) if diag is not None else None))


def load(path, device=None, ctx: Optional[Context] = None):
    """rbd.load (bindings.cpp:80-85) -> read_model (io.cpp:574-622): returns
    (Model, eps_r). device=None: numpy Y/T; a CUDA device: Y/T are torch tensors
    filled straight from the file through pinned staging buffers. `selected` is
    not part of the container (io.hpp:56) and comes back empty."""
    lib = load_library()
    p = os.fsencode(str(path))
    m, n, d = C.c_int64(), C.c_int64(), C.c_int64()
    kind = C.c_int()
    check(lib.rbd_model_read_header(p, C.byref(m), C.byref(n), C.byref(d), C.byref(kind)))
    m, n, d, kind = m.value, n.value, d.value, kind.value
    hist = np.zeros(d)
    diag = np.zeros(m) if kind == 1 else None
    eps = C.c_double()
    if device is not None:
        dev = torch.device(device)
        ctx = ctx or default_context(dev.index or 0)
        Y = torch.empty((d, m), dtype=torch.float64, device=dev).t()
        T = torch.empty((d, n), dtype=torch.float64, device=dev)
        torch.cuda.current_stream(dev).synchronize()
        ldy = m
    else:
        Y = np.zeros((m, d), order="F")
        T = np.zeros((d, n))
        ldy = m
    check(lib.rbd_model_read(ctx.handle if ctx is not None else None, p, _ptr(Y), ldy, _ptr(T),
                             C.byref(eps), _dp(hist), _dp(diag) if diag is not None else None))
    res = Result()
    res.d = d
    return Model(Y, T, d, [], hist, res, ctx, kind, diag), eps.value


class Classifier:
    """rbd::Classifier (classify.hpp:14-21): nearest-neighbour recognition in reduced
    coordinates. ``train_coords`` is ``model.T`` (d x n_train); ``labels`` has one
    entry per training column. Predictions run batched on the GPU
    (rbd_classify_batch: K5 projection + the fused nearest-column kernel)."""

    def __init__(self, model: Model, labels):
        self.model = model
        self.labels = list(labels)
        self._dev = None

    @property
    def train_coords(self):
        return self.model.T

    def _device_model(self):
        if self._dev is None:
            Y, T = self.model.Y, self.model.T
            if _is_torch_cuda(Y):
                Yd = Y if Y.stride(0) == 1 else Y.t().contiguous().t()
                Td = T.contiguous()
            else:
                m, d = Y.shape
                Yd = torch.empty((d, m), dtype=torch.float64, device="cuda").t()
                Yd.copy_(torch.from_numpy(np.asfortranarray(Y)))
                Td = torch.from_numpy(np.ascontiguousarray(T)).cuda()
            torch.cuda.current_stream(Yd.device).synchronize()
            self._dev = (Yd, Td)
        return self._dev

    def predict_indices(self, queries):
        """Best training column per query column (classify.cpp:22-32, batched)."""
        lib = load_library()
        Yd, Td = self._device_model()
        m, d = Yd.shape
        if _is_torch_cuda(queries):
            Qd = queries.reshape(m, -1) if queries.dim() == 1 else queries
            if Qd.dim() != 2 or Qd.shape[0] != m:
                raise DimensionMismatch("project: vector length != m")
            Qd = Qd if Qd.stride(0) == 1 else Qd.t().contiguous().t()
        else:
            qa = np.asarray(queries, dtype=np.float64)
            qa = qa.reshape(-1, 1) if qa.ndim == 1 else qa
            if qa.shape[0] != m:
                raise DimensionMismatch("project: vector length != m")
            Qd = torch.empty((qa.shape[1], m), dtype=torch.float64, device=Yd.device).t()
            Qd.copy_(torch.from_numpy(np.asfortranarray(qa)))
        nq = Qd.shape[1]
        best = torch.empty(nq, dtype=torch.int64, device=Yd.device)
        ctx = self.model._ctx or default_context(Yd.device.index or 0)
        torch.cuda.current_stream(Yd.device).synchronize()
        ldq = Qd.stride(1) if nq > 1 else m
        check(lib.rbd_classify_batch(ctx.handle, C.c_void_p(Yd.data_ptr()), m, d, Yd.stride(1)
                                     if d > 1 else m, C.c_void_p(Td.data_ptr()), Td.shape[1],
                                     C.c_void_p(Qd.data_ptr()), nq, ldq,
                                     C.c_void_p(best.data_ptr()), None))
        ctx.synchronize()
        return best.cpu().numpy()

    def predict(self, v):
        """Classifier::predict (classify.cpp:22-34): the label of the nearest column."""
        return self.labels[int(self.predict_indices(v)[0])]

    def predict_batch(self, queries):
        return [self.labels[int(j)] for j in self.predict_indices(queries)]

    def evaluate(self, test, labels):
        """Fraction of misclassified test columns (classify.cpp:36-48)."""
        ncols = test.shape[1]
        if len(labels) != ncols:
            raise DimensionMismatch("evaluate: one label per test column required")
        if test.shape[0] != self.model.Y.shape[0]:
            raise DimensionMismatch("evaluate: test dimension != training dimension")
        pred = self.predict_batch(test)
        wrong = sum(1 for p_, t_ in zip(pred, labels) if p_ != t_)
        return wrong / ncols


def fit(train, labels, d_max: int, eps_r: float = 0.0, diag=None, sparse=None,
        start_column: int = 0, reorthogonalize: bool = False, ctx: Optional[Context] = None):
    """rbd.fit (bindings.cpp:165-178) -> rbd::fit (classify.cpp:11-20)."""
    labels = list(labels)
    if len(labels) != train.shape[1]:
        raise DimensionMismatch("fit: one label per training column required")
    model = decompose(train, d_max, eps_r, diag=diag, sparse=sparse, start_column=start_column,
                      reorthogonalize=reorthogonalize, ctx=ctx)
    return Classifier(model, labels)


def project(model: Model, v):
    """rbd::project (decompose.cpp:113-117): c = Y'v; DimensionMismatch if len(v) != m."""
    lib = load_library()
    ctx = model._ctx
    if model.on_device:
        vv = v if _is_torch_cuda(v) else torch.as_tensor(np.asarray(v, dtype=np.float64),
                                                          device=model._Y.device)
        vv = vv.reshape(-1).to(torch.float64).contiguous()
        m = model._Y.shape[0]
        if vv.numel() != m:
            raise DimensionMismatch("project: vector length != m")
        out = torch.empty(model.d, dtype=torch.float64, device=vv.device)
        torch.cuda.current_stream(vv.device).synchronize()
        check(lib.rbd_project_batch(ctx.handle, C.c_void_p(model._Y.data_ptr()), m, model.d,
                                    model._Y.stride(1), C.c_void_p(vv.data_ptr()), 1, m,
                                    C.c_void_p(out.data_ptr()), None))
        ctx.synchronize()
        return out
    vv = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))
    if vv.shape[0] != model.Y.shape[0]:
        raise DimensionMismatch("project: vector length != m")
    return model.resident().project(vv.reshape(-1, 1), with_error=False)[0][:, 0]


def reconstruct(model: Model, c):
    """rbd::reconstruct (decompose.cpp:119-123): Y c; DimensionMismatch if len(c) != d."""
    lib = load_library()
    ctx = model._ctx
    if model.on_device:
        cc = c if _is_torch_cuda(c) else torch.as_tensor(np.asarray(c, dtype=np.float64),
                                                          device=model._Y.device)
        cc = cc.reshape(-1).to(torch.float64).contiguous()
        if cc.numel() != model.d:
            raise DimensionMismatch("reconstruct: coefficient length != d")
        m = model._Y.shape[0]
        out = torch.empty(m, dtype=torch.float64, device=cc.device)
        torch.cuda.current_stream(cc.device).synchronize()
        check(lib.rbd_reconstruct(ctx.handle, C.c_void_p(model._Y.data_ptr()), m, model.d,
                                  model._Y.stride(1), C.c_void_p(cc.data_ptr()),
                                  C.c_void_p(out.data_ptr())))
        ctx.synchronize()
        return out
    cc = np.ascontiguousarray(np.asarray(c, dtype=np.float64).reshape(-1))
    if cc.shape[0] != model.d:
        raise DimensionMismatch("reconstruct: coefficient length != d")
    return model.resident().reconstruct(cc.reshape(-1, 1))[:, 0]


class ResidentModel:
    """A model resident in HBM (rbd_model_t): Y (m x d) and T
    (d x n) uploaded once (or read from an RBD1 file straight into HBM); the
    out-of-sample calls move only their own vectors. Host numpy in, host numpy
    out (the reference-facing entries rbd_project_model /
    rbd_project_host_many[_f32] / rbd_reconstruct_model)."""

    def __init__(self, handle, ctx: Context):
        self.handle = handle
        self.ctx = ctx
        self._lib = load_library()
        m, n, d = C.c_int64(), C.c_int64(), C.c_int64()
        eps = C.c_double()
        kind = C.c_int()
        check(self._lib.rbd_model_info(handle, C.byref(m), C.byref(n), C.byref(d), None, None,
                                       C.byref(eps), C.byref(kind)))
        self.m, self.n, self.d = m.value, n.value, d.value
        self.eps_r, self.weight_kind = eps.value, kind.value

    @classmethod
    def from_model(cls, model: "Model", ctx: Optional[Context] = None) -> "ResidentModel":
        lib = load_library()
        Y, T = model.Y, model.T
        h = C.c_void_p()
        hist = np.ascontiguousarray(np.asarray(model.residual_history, dtype=np.float64))
        if _is_torch_cuda(Y):
            ctx = ctx or default_context(Y.device.index or 0)
            Yc = Y if Y.stride(0) == 1 else Y.t().contiguous().t()
            Tc = T.contiguous()
            torch.cuda.current_stream(Y.device).synchronize()
            ldy = Yc.stride(1) if Yc.shape[1] > 1 else Yc.shape[0]
            check(lib.rbd_model_create(ctx.handle, Yc.shape[0], Tc.shape[1], model.d,
                                       C.c_void_p(Yc.data_ptr()), ldy, C.c_void_p(Tc.data_ptr()), 1,
                                       _dp(hist) if hist.size else None, 0.0, C.byref(h)))
        else:
            ctx = ctx or default_context(0)
            Yh = np.asfortranarray(Y, dtype=np.float64)
            Th = np.ascontiguousarray(T, dtype=np.float64)
            check(lib.rbd_model_create(ctx.handle, Yh.shape[0], Th.shape[1], model.d, _dp(Yh),
                                       Yh.shape[0], _dp(Th), 0, _dp(hist) if hist.size else None,
                                       0.0, C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def load(cls, path, ctx: Optional[Context] = None) -> "ResidentModel":
        """read_model (io.cpp:574-622) straight into HBM."""
        ctx = ctx or default_context(0)
        h = C.c_void_p()
        check(load_library().rbd_model_load(ctx.handle, os.fsencode(str(path)), C.byref(h)))
        return cls(h, ctx)

    def close(self):
        if getattr(self, "handle", None):
            self._lib.rbd_model_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def history(self):
        out = np.zeros(self.d)
        check(self._lib.rbd_model_read_vectors(self.handle, _dp(out), None))
        return out

    def device_arrays(self):
        """(Y, T) as torch CUDA views of the resident buffers (no copy)."""
        dy, dt = C.c_void_p(), C.c_void_p()
        check(self._lib.rbd_model_info(self.handle, None, None, None, C.byref(dy), C.byref(dt),
                                       None, None))
        dev = torch.device("cuda", self.ctx.device if hasattr(self.ctx, "device") else 0)
        Y = _torch_from_ptr(dy.value, (self.d, self.m), dev).t()
        T = _torch_from_ptr(dt.value, (self.d, self.n), dev)
        return Y, T

    def _check_x(self, Xn, dtype):
        xa = np.asarray(Xn, dtype=dtype)
        xa = xa.reshape(-1, 1) if xa.ndim == 1 else xa
        if xa.ndim != 2 or xa.shape[0] != self.m:
            raise DimensionMismatch("project: vector length != m")
        return xa if xa.flags["F_CONTIGUOUS"] else np.asfortranarray(xa)

    def project(self, Xn, with_error: bool = True):
        """T_new = Y'X_new (d x N) and err (Eq. 3) for host columns X_new (m x N)."""
        xa = self._check_x(Xn, np.float64)
        N = xa.shape[1]
        Tn = np.zeros((self.d, N), order="F")
        err = np.zeros(N) if with_error else None
        check(self._lib.rbd_project_model(self.ctx.handle, self.handle, _dp(xa), N,
                                          max(self.m, xa.strides[1] // 8 if N > 1 else self.m),
                                          _dp(Tn), _dp(err) if with_error else None))
        return Tn, err

    def project_many(self, batches, with_error: bool = True, f32: bool = False, out=None):
        """A stream of equally sized host batches (rbd_project_host_many[_f32]):
        the upload of batch i+1 overlaps the contraction of batch i. Page-locked
        batches (e.g. torch.empty(..., pin_memory=True).numpy()) are needed for
        the overlap. Returns [(T_new, err)] per batch; `out` may pass
        preallocated (T_new, err) pairs (page-locked outputs download during
        the stream)."""
        dt = np.float32 if f32 else np.float64
        xs = [self._check_x(b, dt) for b in batches]
        if not xs:
            return []
        N = xs[0].shape[1]
        if any(x.shape != xs[0].shape or x.strides != xs[0].strides for x in xs):
            raise InvalidArgument("project_many: batches must share one shape and layout")
        ldx = xs[0].strides[1] // xs[0].itemsize if N > 1 else self.m
        cnt = len(xs)
        if out is None:
            out = [(np.zeros((self.d, N), dtype=dt, order="F"),
                    np.zeros(N) if with_error else None) for _ in range(cnt)]
        P = C.c_void_p * cnt
        xp = P(*[x.ctypes.data for x in xs])
        tp = P(*[o[0].ctypes.data for o in out])
        ep = P(*[(o[1].ctypes.data if o[1] is not None else None) for o in out])
        fn = self._lib.rbd_project_host_many_f32 if f32 else self._lib.rbd_project_host_many
        check(fn(self.ctx.handle, self.handle, cnt, xp, N, ldx, tp, ep if with_error else None))
        return out

    def reconstruct(self, Cm):
        """V = Y C for host coefficients C (d x N)."""
        ca = np.asfortranarray(np.asarray(Cm, dtype=np.float64))
        ca = ca.reshape(-1, 1) if ca.ndim == 1 else ca
        if ca.shape[0] != self.d:
            raise DimensionMismatch("reconstruct: coefficient length != d")
        V = np.zeros((self.m, ca.shape[1]), order="F")
        check(self._lib.rbd_reconstruct_model(self.ctx.handle, self.handle, _dp(ca), ca.shape[1],
                                              _dp(V)))
        return V


def _torch_from_ptr(addr, shape, device):
    """A torch float64 view of `shape` on raw device memory owned elsewhere."""
    n = int(np.prod(shape))

    class _Cai:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (addr, False),
                                    "version": 3, "strides": None}
    t = torch.as_tensor(_Cai(), device=device)
    assert t.numel() == n
    return t


def project_batch(Y, Xn, with_error: bool = True, ctx: Optional[Context] = None):
    """Batched out-of-sample compression: T_new = Y'X_new (d x N) and the identity
    error indicator err_j = max(||x_j||^2 - ||t_j||^2, 0) (Eq. 3). Device tensors
    (column-major views) or numpy arrays."""
    lib = load_library()
    if _is_torch_cuda(Y):
        ctx = ctx or default_context(Y.device.index or 0)
        Yc, ldy = _col_major_torch(Y)
        Xc, ldx = _col_major_torch(Xn)
        m, d = Yc.shape
        if Xc.shape[0] != m:
            raise DimensionMismatch("project: vector length != m")
        N = Xc.shape[1]
        Tn = torch.empty((N, d), dtype=torch.float64, device=Y.device).t()
        err = torch.empty(N, dtype=torch.float64, device=Y.device) if with_error else None
        ldt = Tn.stride(1)
        assert ldt == d
        torch.cuda.current_stream(Y.device).synchronize()
        check(lib.rbd_project_batch(ctx.handle, C.c_void_p(Yc.data_ptr()), m, d, ldy,
                                    C.c_void_p(Xc.data_ptr()), N, ldx, C.c_void_p(Tn.data_ptr()),
                                    C.c_void_p(err.data_ptr()) if err is not None else None))
        ctx.synchronize()
        return Tn, err
    ctx = ctx or default_context(0)
    Ya = _col_major_np(Y)
    Xa = _col_major_np(Xn)
    m, d = Ya.shape
    if Xa.shape[0] != m:
        raise DimensionMismatch("project: vector length != m")
    N = Xa.shape[1]
    Tn = np.zeros((d, N), dtype=np.float64, order="F")
    err = np.zeros(N, dtype=np.float64)
    check(lib.rbd_project_host(ctx.handle, _dp(Ya), m, d, _dp(Xa), N, _dp(Tn),
                               _dp(err) if with_error else None))
    return Tn, (err if with_error else None)


def project_batch_f32(Y, Xn, with_error: bool = True, ctx: Optional[Context] = None):
    """fp32 mode of the out-of-sample compression: Y, X_new as float32 CUDA
    tensors (column-major views, leading dimensions multiple of 4); T_new on the
    tcgen05 tensor cores (3xTF32), error indicator accumulated in fp64."""
    lib = load_library()
    if not (_is_torch_cuda(Y) and _is_torch_cuda(Xn)):
        raise InvalidArgument("project_batch_f32: pass torch CUDA tensors")
    ctx = ctx or default_context(Y.device.index or 0)

    def colmajor32(a):
        a = a.to(torch.float32)
        m_ = a.shape[0]
        if a.stride(0) == 1 and a.stride(1) >= m_ and a.stride(1) % 4 == 0:
            return a, a.stride(1)
        ld = (m_ + 3) // 4 * 4
        buf = torch.zeros((a.shape[1], ld), dtype=torch.float32, device=a.device)
        buf[:, :m_] = a.t()
        return buf.t()[:m_], ld
    Yc, ldy = colmajor32(Y)
    Xc, ldx = colmajor32(Xn)
    m, d = Yc.shape
    if Xc.shape[0] != m:
        raise DimensionMismatch("project: vector length != m")
    N = Xc.shape[1]
    Tn = torch.empty((N, d), dtype=torch.float32, device=Y.device).t()
    err = torch.empty(N, dtype=torch.float64, device=Y.device) if with_error else None
    torch.cuda.current_stream(Y.device).synchronize()
    check(lib.rbd_project_batch_f32(ctx.handle, C.c_void_p(Yc.data_ptr()), m, d, ldy,
                                    C.c_void_p(Xc.data_ptr()), N, ldx, C.c_void_p(Tn.data_ptr()),
                                    C.c_void_p(err.data_ptr()) if err is not None else None))
    ctx.synchronize()
    return Tn, err


def mgs_project(v, basis, breakdown_tol: float, reorthogonalize: bool = False,
                ctx: Optional[Context] = None):
    """rbd::mgs_project (decompose.cpp:12-33) on device tensors.

    Returns (xi, residual_norm) or None on breakdown (std::nullopt).
    ``basis`` is an m x k column-major CUDA tensor (k may be 0)."""
    if not _is_torch_cuda(v):
        raise InvalidArgument("mgs_project: pass torch CUDA tensors (device entry point)")
    lib = load_library()
    ctx = ctx or default_context(v.device.index or 0)
    vv = v.reshape(-1).to(torch.float64).contiguous()
    m = vv.numel()
    if basis is None or basis.numel() == 0:
        k, ldb, bptr = 0, m, None
    else:
        B, ldb = _col_major_torch(basis)
        if B.shape[0] != m:
            raise DimensionMismatch("mgs_project: vector length != basis row count")
        k, bptr = B.shape[1], C.c_void_p(B.data_ptr())
    xi = torch.empty(m, dtype=torch.float64, device=v.device)
    norm = C.c_double()
    ok = C.c_int()
    torch.cuda.current_stream(v.device).synchronize()
    check(lib.rbd_mgs_project(ctx.handle, C.c_void_p(vv.data_ptr()), m, bptr, k, ldb,
                              float(breakdown_tol), 1 if reorthogonalize else 0,
                              C.c_void_p(xi.data_ptr()), C.byref(norm), C.byref(ok)))
    if not ok.value:
        return None
    return xi, norm.value


class Workspace:
    """ErrorWorkspace (workspace.hpp:18-30) on device, identity or diagonal weight.

    workspace_init (workspace.cpp:9-41) at construction; extend(xi)
    (workspace.cpp:43-79); scan() (identity, workspace.cpp:101-113,123) and
    scan_T(T) (any weight, :101-125); error_sq(j, c) (workspace.cpp:84-99)."""

    def __init__(self, x, cap: Optional[int] = None, ctx: Optional[Context] = None, diag=None):
        if not _is_torch_cuda(x):
            raise InvalidArgument("Workspace: pass a torch CUDA tensor")
        self._lib = load_library()
        self.ctx = ctx or default_context(x.device.index or 0)
        self._x, ldx = _col_major_torch(x)
        self.m, self.n = self._x.shape
        self.cap = cap if cap is not None else self.n
        h = C.c_void_p()
        torch.cuda.current_stream(x.device).synchronize()
        if diag is None:
            self.weight_kind = 0
            check(self._lib.rbd_ws_init(self.ctx.handle, C.c_void_p(self._x.data_ptr()), self.m,
                                        self.n, ldx, self.cap, C.byref(h)))
        else:   # WeightSpec::diagonal (workspace.cpp:24-29)
            self.weight_kind = 1
            self._diag = torch.as_tensor(diag, dtype=torch.float64,
                                         device=x.device).reshape(-1).contiguous()
            torch.cuda.current_stream(x.device).synchronize()
            check(self._lib.rbd_ws_init_diag(
                self.ctx.handle, C.c_void_p(self._x.data_ptr()), self.m, self.n, ldx, self.cap,
                C.c_void_p(self._diag.data_ptr()) if self._diag.numel() else None,
                self._diag.numel(), C.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            self._lib.rbd_ws_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def d(self) -> int:
        return int(self._lib.rbd_ws_d(self.handle))

    def extend(self, xi):
        xv = xi.reshape(-1).to(torch.float64).contiguous()
        if xv.numel() != self.m:
            raise DimensionMismatch("workspace_extend: dimensions changed since init")
        torch.cuda.current_stream(xv.device).synchronize()
        check(self._lib.rbd_ws_extend(self.handle, C.c_void_p(xv.data_ptr())))

    def scan(self):
        e = C.c_double()
        j = C.c_int64()
        check(self._lib.rbd_ws_scan(self.handle, C.byref(e), C.byref(j)))
        return e.value, j.value

    def scan_T(self, T):
        """residual_scan(ws, T) for any weight: T is d x n (numpy or CUDA tensor)."""
        e = C.c_double()
        j = C.c_int64()
        if _is_torch_cuda(T):
            Tc = T.contiguous()
            torch.cuda.current_stream(T.device).synchronize()
            check(self._lib.rbd_ws_scan_T(self.handle, C.c_void_p(Tc.data_ptr()), C.byref(e),
                                          C.byref(j)))
        else:
            Th = np.ascontiguousarray(np.asarray(T, dtype=np.float64))
            if Th.shape != (self.d, self.n):
                raise DimensionMismatch("residual_scan: T shape does not match workspace")
            check(self._lib.rbd_ws_scan_T_host(self.handle, _dp(Th) if Th.size else None,
                                               C.byref(e), C.byref(j)))
        return e.value, j.value

    def yay(self):
        """Y'AY (d x d) of a diagonal workspace (workspace.cpp:69-75)."""
        out = np.zeros((max(self.d, 1), max(self.d, 1)))
        check(self._lib.rbd_ws_read_yay(self.handle, _dp(out)))
        return out[: self.d, : self.d]

    def error_sq(self, j: int, c) -> float:
        cc = np.ascontiguousarray(np.asarray(c, dtype=np.float64).reshape(-1))
        out = C.c_double()
        check(self._lib.rbd_ws_error_sq(self.handle, int(j), _dp(cc) if cc.size else None,
                                        cc.shape[0], C.byref(out)))
        return out.value

    def read(self):
        col_sq = np.zeros(self.n)
        resid = np.zeros(self.n)
        yax = np.zeros((max(self.d, 1), self.n))
        check(self._lib.rbd_ws_read(self.handle, _dp(col_sq), _dp(resid), _dp(yax)))
        return col_sq, resid, yax[: self.d]
