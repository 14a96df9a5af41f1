// rbd_ws.cu — the ErrorWorkspace API (proj/include/rbd/workspace.hpp:18-54,
// workspace.cpp:9-125) behind the C ABI: identity and diagonal weights, device
// and host entries.
#include "rbd_capi_internal.h"
#include "rbd_weighted.cuh"

extern "C" {

// ---------------------------------------------------------------------------
// Workspace API
// ---------------------------------------------------------------------------
int rbd_ws_init(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx, int64_t cap,
                rbd_ws_t* out) {
  if (!ctx || !out) return set_err(RBD_ERR_INVALID_ARGUMENT, "null argument");
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "workspace_init: empty matrix");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "workspace_init: ldx < m");
  CU(cudaSetDevice(ctx->device));
  auto* ws = new rbd_ws_s();
  ws->ctx = ctx;
  ws->X = dX;
  ws->m = m;
  ws->n = n;
  ws->ldx = ldx;
  ws->cap = std::max<int64_t>(cap, 1);
  ws->d = 0;
  const long long S = cdiv(m, kChunk);
  int rc = RBD_OK;
  if ((rc = ensure(ws->T, sizeof(double) * ws->cap * n)) ||
      (rc = ensure(ws->colsq, sizeof(double) * n)) || (rc = ensure(ws->resid, sizeof(double) * n)) ||
      (rc = ensure(ws->partial, sizeof(double) * S * n)) ||
      (rc = ensure(ws->rec, sizeof(Rec) * (size_t)ctx->nsm * 8)) ||
      (rc = ensure(ws->counter, 64)) || (rc = ensure(ws->out, 64)) ||
      (rc = ensure(ws->tmp, sizeof(DevState) + 64))) {
    rbd_ws_destroy(ws);
    return rc;
  }
  cudaMemsetAsync(ws->counter.p, 0, 64, ctx->stream);
  cudaMemsetAsync(ws->tmp.p, 0, sizeof(DevState), ctx->stream);
  rc = enqueue_init(ctx, dX, m, n, ldx, ptr<double>(ws->partial), ptr<double>(ws->colsq),
                    ptr<double>(ws->resid), ptr<DevState>(ws->tmp));
  if (rc == RBD_OK && cudaStreamSynchronize(ctx->stream) != cudaSuccess)
    rc = set_err(RBD_ERR_CUDA, "workspace_init: kernel failure");
  if (rc != RBD_OK) {
    rbd_ws_destroy(ws);
    return rc;
  }
  *out = ws;
  return RBD_OK;
}

int rbd_ws_destroy(rbd_ws_t ws) {
  if (!ws) return RBD_OK;
  DevBuf* bl[] = {&ws->T,       &ws->colsq, &ws->resid, &ws->partial, &ws->rec,
                  &ws->counter, &ws->out,   &ws->tmp,   &ws->Xown,    &ws->diag,
                  &ws->basis,   &ws->axi,   &ws->yy,    &ws->yay,     &ws->row};
  for (DevBuf* b : bl) release(*b);
  delete ws;
  return RBD_OK;
}

int64_t rbd_ws_d(rbd_ws_t ws) { return ws ? ws->d : 0; }

int rbd_ws_extend(rbd_ws_t ws, const double* dxi) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  if (ws->d >= ws->cap) return set_err(RBD_ERR_INVALID_ARGUMENT, "workspace_extend: capacity exhausted");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  if (ws->kind == 1) {   // diagonal, workspace.cpp:61-79
    const long long m = ws->m, n = ws->n, d = ws->d, S = cdiv(m, kChunk);
    double* basis = ptr<double>(ws->basis);
    CU(cudaMemcpyAsync(basis + d * m, dxi, sizeof(double) * m, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    // a o xi (weight.cpp:83) and xi'A xi (:75): k_diag_vec reads column st->d of
    // its "Y" argument; the workspace's scratch state has d = 0, done = 0
    DevState* st0 = ptr<DevState>(ws->tmp);
    const int gv = diag_vec_grid(ctx, m);
    k_diag_vec<<<gv, kThreads, 0, ctx->stream>>>(basis + d * m, m, ptr<double>(ws->diag),
                                                 ptr<double>(ws->axi), ptr<double>(ws->yy), st0);
    ctx->launches++;
    // YAX row d = X'(a o xi) (:66)
    const int vx = (ws->ldx % 2 == 0 && aligned16(ws->X) && aligned16(ws->axi.p)) ? 2 : 1;
    SweepArgs s{};
    s.A = ws->X;
    s.lda = ws->ldx;
    s.m = m;
    s.ncols = n;
    s.v = ptr<double>(ws->axi);
    s.partial = ptr<double>(ws->partial);
    s.pstride = n;
    s.gate = GATE_NONE;
    TRY(launch_sweep(ctx, s, vx, MODE_DOT, true, n));
    const int gr = (int)std::max<long long>(1, std::min<long long>(cdiv(n, 256), (long long)ctx->nsm * 4));
    k_rowsum<<<gr, 256, 0, ctx->stream>>>(ptr<double>(ws->partial), S, n, ptr<double>(ws->T) + d * n);
    ctx->launches++;
    // YAY row d (:69-75): the earlier basis vectors against a o xi
    if (d > 0) {
      const int vb = (m % 2 == 0 && aligned16(ws->basis.p) && aligned16(ws->axi.p)) ? 2 : 1;
      SweepArgs b{};
      b.A = basis;
      b.lda = m;
      b.m = m;
      b.ncols = d;
      b.v = ptr<double>(ws->axi);
      b.partial = ptr<double>(ws->partial);
      b.pstride = d;
      b.gate = GATE_NONE;
      TRY(launch_sweep(ctx, b, vb, MODE_DOT, false, d));
      k_rowsum<<<(unsigned)std::max<long long>(1, cdiv(d, 256)), 256, 0, ctx->stream>>>(
          ptr<double>(ws->partial), S, d, ptr<double>(ws->row));
      ctx->launches++;
    }
    k_yay_row<<<(unsigned)std::max<long long>(1, cdiv(d, 256)), 256, 0, ctx->stream>>>(
        ptr<double>(ws->row), d, ptr<double>(ws->yy), gv, ptr<double>(ws->yay), ws->cap);
    ctx->launches++;
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(ctx->stream));
    ws->d += 1;
    return RBD_OK;
  }
  const int vec = (ws->ldx % 2 == 0 && aligned16(ws->X) && aligned16(dxi)) ? 2 : 1;
  SweepArgs s{};
  s.A = ws->X;
  s.lda = ws->ldx;
  s.m = ws->m;
  s.ncols = ws->n;
  s.v = dxi;
  s.partial = ptr<double>(ws->partial);
  s.pstride = ws->n;
  s.st = nullptr;
  s.gate = GATE_NONE;
  TRY(launch_sweep(ctx, s, vec, MODE_DOT, true, ws->n));
  FinalizeArgs f{};
  f.partial = ptr<double>(ws->partial);
  f.S = cdiv(ws->m, kChunk);
  f.n = ws->n;
  f.T = ptr<double>(ws->T);
  f.krow = ws->d;
  f.r = ptr<double>(ws->resid);
  f.col_sq = ptr<double>(ws->colsq);
  f.st = nullptr;
  f.mode = 1;
  k_finalize<<<finalize_grid(ctx, ws->n), kThreads, 0, ctx->stream>>>(f);
  ctx->launches++;
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(ctx->stream));
  ws->d += 1;
  return RBD_OK;
}

int rbd_ws_scan(rbd_ws_t ws, double* e_cur, int64_t* argmax) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  const int g = finalize_grid(ctx, ws->n);
  k_scan_only<<<g, kThreads, 0, ctx->stream>>>(ptr<double>(ws->resid), ws->n, ptr<Rec>(ws->rec),
                                                ptr<unsigned>(ws->counter), ptr<Rec>(ws->out));
  ctx->launches++;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(ctx->h_rec, ws->out.p, sizeof(Rec), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (e_cur) *e_cur = ctx->h_rec->v;
  if (argmax) *argmax = ctx->h_rec->j;
  return RBD_OK;
}

int rbd_ws_error_sq(rbd_ws_t ws, int64_t j, const double* h_c, int64_t clen, double* out) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  if (j < 0 || j >= ws->n) return set_err(RBD_ERR_INDEX_OUT_OF_RANGE, "error_sq: column index out of range");
  if (clen != ws->d) return set_err(RBD_ERR_DIMENSION_MISMATCH, "error_sq: coefficient length != d");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  double* dc = reinterpret_cast<double*>(static_cast<char*>(ws->tmp.p) + sizeof(DevState));
  DevBuf cbuf;
  if (clen > 0) {
    TRY(ensure(cbuf, sizeof(double) * clen));
    CU(cudaMemcpyAsync(cbuf.p, h_c, sizeof(double) * clen, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (ws->kind == 1)
    k_error_sq_w<<<1, kThreads, 0, ctx->stream>>>(ptr<double>(ws->T), ws->n, ws->d, j,
                                                  ptr<double>(cbuf), ptr<double>(ws->yay), ws->cap,
                                                  ptr<double>(ws->colsq), dc);
  else
    k_error_sq<<<1, kThreads, 0, ctx->stream>>>(ptr<double>(ws->T), ws->n, ws->d, j,
                                                ptr<double>(cbuf), ptr<double>(ws->colsq), dc);
  ctx->launches++;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(out, dc, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  release(cbuf);
  return RBD_OK;
}

int rbd_ws_read(rbd_ws_t ws, double* h_col_sq, double* h_residual_sq, double* h_yax) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  if (h_col_sq) CU(cudaMemcpyAsync(h_col_sq, ws->colsq.p, sizeof(double) * ws->n, cudaMemcpyDeviceToHost, ctx->stream));
  if (h_residual_sq)
    CU(cudaMemcpyAsync(h_residual_sq, ws->resid.p, sizeof(double) * ws->n, cudaMemcpyDeviceToHost, ctx->stream));
  if (h_yax && ws->d > 0)
    CU(cudaMemcpyAsync(h_yax, ws->T.p, sizeof(double) * ws->d * ws->n, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return RBD_OK;
}

int rbd_ws_init_diag(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx,
                     int64_t cap, const double* d_diag, int64_t diag_len, rbd_ws_t* out) {
  if (!ctx || !out) return set_err(RBD_ERR_INVALID_ARGUMENT, "null argument");
  CU(cudaSetDevice(ctx->device));
  std::vector<double> h((size_t)std::max<int64_t>(diag_len, 0));
  if (diag_len > 0) {
    if (!d_diag) return set_err(RBD_ERR_INVALID_ARGUMENT, "workspace_init: null diagonal");
    CU(cudaMemcpyAsync(h.data(), d_diag, sizeof(double) * diag_len, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  TRY(check_diagonal(h.data(), diag_len));                              // weight.cpp:11-17
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "workspace_init: empty matrix");
  if (diag_len != m)                                                    // workspace.cpp:12-13
    return set_err(RBD_ERR_INCOMPATIBLE_WEIGHT, "weight dimension does not match matrix rows");
  rbd_ws_t ws = nullptr;
  TRY(rbd_ws_init(ctx, dX, m, n, ldx, cap, &ws));
  int rc = RBD_OK;
  const long long c = ws->cap;
  if ((rc = ensure(ws->diag, sizeof(double) * m)) || (rc = ensure(ws->basis, sizeof(double) * m * c)) ||
      (rc = ensure(ws->axi, sizeof(double) * m)) ||
      (rc = ensure(ws->yy, sizeof(double) * diag_vec_grid(ctx, m))) ||
      (rc = ensure(ws->yay, sizeof(double) * c * c)) ||
      (rc = ensure(ws->row, sizeof(double) * std::max<long long>(c, 1))) ||
      (rc = ensure(ws->partial, sizeof(double) * cdiv(m, kChunk) * std::max<long long>(n, c)))) {
    rbd_ws_destroy(ws);
    return rc;
  }
  ws->kind = 1;
  cudaMemcpyAsync(ws->diag.p, d_diag, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream);
  cudaMemsetAsync(ws->yay.p, 0, sizeof(double) * c * c, ctx->stream);
  // col_sq = diag(X'AX) (workspace.cpp:24-29), residual_sq = col_sq (:38)
  const int g = (int)std::max<long long>(1, std::min<long long>(n, (long long)ctx->nsm * 8));
  k_colsq_diag<<<g, kThreads, 0, ctx->stream>>>(dX, ldx, m, n, ptr<double>(ws->diag),
                                                ptr<double>(ws->colsq));
  ctx->launches++;
  cudaMemcpyAsync(ws->resid.p, ws->colsq.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream);
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    rbd_ws_destroy(ws);
    return set_err(RBD_ERR_CUDA, "workspace_init: kernel failure");
  }
  *out = ws;
  return RBD_OK;
}

int rbd_ws_scan_T(rbd_ws_t ws, const double* dT, double* e_cur, int64_t* argmax) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  if (ws->d > 0 && !dT) return set_err(RBD_ERR_DIMENSION_MISMATCH, "residual_scan: T shape does not match workspace");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  const int g = finalize_grid(ctx, ws->n);
  k_scan_T<<<g, kThreads, 0, ctx->stream>>>(ptr<double>(ws->T), dT, ws->n, ws->d,
                                            ws->kind == 1 ? ptr<double>(ws->yay) : nullptr, ws->cap,
                                            ptr<double>(ws->colsq), ptr<Rec>(ws->rec),
                                            ptr<unsigned>(ws->counter), ptr<Rec>(ws->out));
  ctx->launches++;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(ctx->h_rec, ws->out.p, sizeof(Rec), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (e_cur) *e_cur = ctx->h_rec->v;
  if (argmax) *argmax = ctx->h_rec->j;
  return RBD_OK;
}

int rbd_ws_scan_T_host(rbd_ws_t ws, const double* hT, double* e_cur, int64_t* argmax) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  DevBuf tb;
  if (ws->d > 0) {
    TRY(ensure(tb, sizeof(double) * ws->d * ws->n));
    if (cudaMemcpyAsync(tb.p, hT, sizeof(double) * ws->d * ws->n, cudaMemcpyHostToDevice,
                        ctx->stream) != cudaSuccess) {
      release(tb);
      return set_err(RBD_ERR_CUDA, "residual_scan: H2D failed");
    }
  }
  const int rc = rbd_ws_scan_T(ws, ws->d > 0 ? ptr<double>(tb) : nullptr, e_cur, argmax);
  release(tb);
  return rc;
}

int rbd_ws_read_yay(rbd_ws_t ws, double* h_yay) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  if (ws->kind != 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "read_yay: identity workspace (Y'AY = I)");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  if (ws->d > 0)
    CU(cudaMemcpy2DAsync(h_yay, sizeof(double) * ws->d, ws->yay.p, sizeof(double) * ws->cap,
                         sizeof(double) * ws->d, ws->d, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return RBD_OK;
}


int rbd_ws_init_host(rbd_ctx_t ctx, const double* hX, int64_t m, int64_t n, int64_t ldx,
                     int64_t cap, rbd_ws_t* out) {
  if (!ctx || !out) return set_err(RBD_ERR_INVALID_ARGUMENT, "null argument");
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "workspace_init: empty matrix");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "workspace_init: ldx < m");
  CU(cudaSetDevice(ctx->device));
  DevBuf xb;
  TRY(ensure(xb, sizeof(double) * m * n));
  if (cudaMemcpy2DAsync(xb.p, sizeof(double) * m, hX, sizeof(double) * ldx, sizeof(double) * m, n,
                        cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess) {
    release(xb);
    return set_err(RBD_ERR_CUDA, "workspace_init: H2D failed");
  }
  rbd_ws_t ws = nullptr;
  int rc = rbd_ws_init(ctx, ptr<double>(xb), m, n, m, cap, &ws);
  if (rc) {
    release(xb);
    return rc;
  }
  ws->Xown = xb;
  *out = ws;
  return RBD_OK;
}

int rbd_ws_init_diag_host(rbd_ctx_t ctx, const double* hX, int64_t m, int64_t n, int64_t ldx,
                          int64_t cap, const double* h_diag, int64_t diag_len, rbd_ws_t* out) {
  if (!ctx || !out) return set_err(RBD_ERR_INVALID_ARGUMENT, "null argument");
  TRY(check_diagonal(h_diag, diag_len));
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "workspace_init: empty matrix");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "workspace_init: ldx < m");
  if (diag_len != m)
    return set_err(RBD_ERR_INCOMPATIBLE_WEIGHT, "weight dimension does not match matrix rows");
  CU(cudaSetDevice(ctx->device));
  DevBuf xb, db;
  TRY(ensure(xb, sizeof(double) * m * n));
  if (ensure(db, sizeof(double) * m) != RBD_OK ||
      cudaMemcpy2DAsync(xb.p, sizeof(double) * m, hX, sizeof(double) * ldx, sizeof(double) * m, n,
                        cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
      cudaMemcpyAsync(db.p, h_diag, sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream) !=
          cudaSuccess) {
    release(xb);
    release(db);
    return set_err(RBD_ERR_CUDA, "workspace_init: H2D failed");
  }
  rbd_ws_t ws = nullptr;
  int rc = rbd_ws_init_diag(ctx, ptr<double>(xb), m, n, m, cap, ptr<double>(db), m, &ws);
  release(db);   // the workspace keeps its own copy of the weight
  if (rc) {
    release(xb);
    return rc;
  }
  ws->Xown = xb;
  *out = ws;
  return RBD_OK;
}

int rbd_ws_extend_host(rbd_ws_t ws, const double* hxi) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  DevBuf& b = ws->ctx->hs[0];   // context scratch, kept between calls
  TRY(ensure(b, sizeof(double) * ws->m));
  // on the workspace's stream (a pageable-source cudaMemcpy may return before its
  // DMA lands, and the context stream does not wait for the legacy stream)
  if (cudaMemcpyAsync(b.p, hxi, sizeof(double) * ws->m, cudaMemcpyHostToDevice,
                      ws->ctx->stream) != cudaSuccess)
    return set_err(RBD_ERR_CUDA, "workspace_extend: H2D failed");
  return rbd_ws_extend(ws, ptr<double>(b));
}

}  // extern "C"
