// rbd_model.cu — device-resident models (SURVEY §8(b) rbd_model_t) and the
// out-of-sample entries that run on them: project (decompose.cpp:113-117) and
// reconstruct (:119-123) with host buffers, and the pipelined batch stream of
// BASELINE config 4 (rbd_project_host_many[_f32]).
//
// The reference's callers apply one finished model to many vectors
// (classify.cpp:22-23 per query, tools/main.cpp:149-158 per column). With Y
// resident in HBM, a call moves only its own vectors: no Y upload, no
// allocation (the context keeps its scratch), no cudaFree device sync.
#include "rbd_capi_internal.h"

struct rbd_model_s {
  int device = 0;
  int64_t m = 0, n = 0, d = 0;
  DevBuf Y, T;          // Y m x d column-major (ld m); T d x n row-major
  DevBuf Y32;           // fp32 copy of Y for K6 (ld ld32, multiple of 4), made on first use
  int64_t ld32 = 0;
  double eps_r = 0.0;
  int weight_kind = 0;
  std::vector<double> history, diag;
};

namespace {

__global__ void k_f64_to_f32_cols(const double* __restrict__ src, long long m, long long cols,
                                  long long lds, float* __restrict__ dst, long long ldd) {
  const long long total = ldd * cols;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long j = t / ldd, i = t - j * ldd;
    dst[t] = i < m ? (float)src[i + j * lds] : 0.0f;
  }
}

int ensure_y32(rbd_ctx_t ctx, rbd_model_t md) {
  if (md->Y32.p) return RBD_OK;
  md->ld32 = (md->m + 3) / 4 * 4;
  TRY(ensure(md->Y32, sizeof(float) * (size_t)md->ld32 * (size_t)md->d));
  k_f64_to_f32_cols<<<1184, 256, 0, ctx->stream>>>(ptr<double>(md->Y), md->m, md->d, md->m,
                                                   ptr<float>(md->Y32), md->ld32);
  ctx->launches++;
  CU(cudaGetLastError());
  return RBD_OK;
}

int check_model(rbd_ctx_t ctx, rbd_model_t md) {
  if (!ctx || !md) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context/model");
  if (ctx->device != md->device)
    return set_err(RBD_ERR_INVALID_ARGUMENT, "model lives on another device than the context");
  return RBD_OK;
}

struct Events {
  cudaEvent_t e[6] = {};
  ~Events() {
    for (cudaEvent_t x : e)
      if (x) cudaEventDestroy(x);
  }
  int create() {
    for (cudaEvent_t& x : e) CU(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    return RBD_OK;
  }
};

// count batches of N columns: upload (up_stream) -> contraction (ctx->stream)
// -> download (d2h_stream), two buffers per operand, ordered by events only.
template <typename TX, typename TT>
int project_stream(rbd_ctx_t ctx, rbd_model_t md, int64_t count, const TX* const* hXn, int64_t N,
                   int64_t ldx, TT* const* hTn, double* const* h_err, bool f32) {
  TRY(check_model(ctx, md));
  if (count < 0 || N < 0) return set_err(RBD_ERR_INVALID_ARGUMENT, "project: bad batch count/size");
  if (count == 0 || N == 0) return RBD_OK;
  if (!hXn) return set_err(RBD_ERR_INVALID_ARGUMENT, "project: null input batches");
  if (ldx < md->m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "project: vector length != m");
  for (int64_t i = 0; i < count; ++i)
    if (!hXn[i]) return set_err(RBD_ERR_INVALID_ARGUMENT, "project: null input batch");
  CU(cudaSetDevice(ctx->device));
  NvtxRange nv(f32 ? "rbd.project_stream_f32" : "rbd.project_stream");
  const int64_t m = md->m, d = md->d;
  if (f32) TRY(ensure_y32(ctx, md));
  const int64_t ldd = f32 ? md->ld32 : m;
  const size_t xb = sizeof(TX) * (size_t)ldd * (size_t)N;
  const size_t tb = sizeof(TT) * (size_t)d * (size_t)N;
  const size_t eb = sizeof(double) * (size_t)N;
  const int nbuf = count > 1 ? 2 : 1;
  for (int b = 0; b < nbuf; ++b) {
    TRY(ensure(ctx->pm_X[b], xb));
    TRY(ensure(ctx->pm_T[b], tb));
    TRY(ensure(ctx->pm_E[b], eb));
  }
  if (f32 && ldd != m) {   // zero rows of the padded columns (TMA reads them)
    for (int b = 0; b < nbuf; ++b) CU(cudaMemsetAsync(ctx->pm_X[b].p, 0, xb, ctx->stream));
  }
  if (!ctx->up_stream) CU(cudaStreamCreateWithFlags(&ctx->up_stream, cudaStreamNonBlocking));
  if (!ctx->d2h_stream) CU(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
  Events ev;
  TRY(ev.create());
  cudaEvent_t* up = ev.e;        // upload of buffer b landed
  cudaEvent_t* comp = ev.e + 2;  // contraction on buffer b done (X read, T/err written)
  cudaEvent_t* down = ev.e + 4;  // T/err of buffer b copied out
  // the memsets / Y32 conversion precede every upload and every contraction
  CU(cudaEventRecord(comp[0], ctx->stream));
  CU(cudaStreamWaitEvent(ctx->up_stream, comp[0], 0));
  auto upload = [&](int64_t i) -> int {
    const int b = (int)(i & 1);
    if (i >= 2) CU(cudaStreamWaitEvent(ctx->up_stream, comp[b], 0));   // batch i-2 read it
    CU(cudaMemcpy2DAsync(ctx->pm_X[b].p, sizeof(TX) * ldd, hXn[i], sizeof(TX) * ldx,
                         sizeof(TX) * m, N, cudaMemcpyHostToDevice, ctx->up_stream));
    CU(cudaEventRecord(up[b], ctx->up_stream));
    return RBD_OK;
  };
  int rc = upload(0);
  for (int64_t i = 0; i < count && rc == RBD_OK; ++i) {
    const int b = (int)(i & 1);
    if (i + 1 < count && (rc = upload(i + 1)) != RBD_OK) break;
    CU(cudaStreamWaitEvent(ctx->stream, up[b], 0));
    if (i >= 2) CU(cudaStreamWaitEvent(ctx->stream, down[b], 0));   // batch i-2's outputs out
    double* de = (h_err && h_err[i]) ? ptr<double>(ctx->pm_E[b]) : nullptr;
    if constexpr (sizeof(TX) == 4)
      rc = rbd_project_batch_f32(ctx, ptr<float>(md->Y32), m, d, md->ld32, ptr<float>(ctx->pm_X[b]),
                                 N, ldd, ptr<float>(ctx->pm_T[b]), de);
    else
      rc = rbd_project_batch(ctx, ptr<double>(md->Y), m, d, m, ptr<double>(ctx->pm_X[b]), N, ldd,
                             ptr<double>(ctx->pm_T[b]), de);
    if (rc != RBD_OK) break;
    CU(cudaEventRecord(comp[b], ctx->stream));
    CU(cudaStreamWaitEvent(ctx->d2h_stream, comp[b], 0));
    if (hTn && hTn[i])
      CU(cudaMemcpyAsync(hTn[i], ctx->pm_T[b].p, tb, cudaMemcpyDeviceToHost, ctx->d2h_stream));
    if (de) CU(cudaMemcpyAsync(h_err[i], de, eb, cudaMemcpyDeviceToHost, ctx->d2h_stream));
    CU(cudaEventRecord(down[b], ctx->d2h_stream));
  }
  // drain all three streams, even after an error, before the buffers are reused
  const cudaError_t e1 = cudaStreamSynchronize(ctx->up_stream);
  const cudaError_t e2 = cudaStreamSynchronize(ctx->stream);
  const cudaError_t e3 = cudaStreamSynchronize(ctx->d2h_stream);
  if (rc != RBD_OK) return rc;
  for (cudaError_t e : {e1, e2, e3})
    if (e != cudaSuccess) return set_err(RBD_ERR_CUDA, std::string("project stream: ") + cudaGetErrorString(e));
  return RBD_OK;
}

}  // namespace

extern "C" {

int rbd_model_create(rbd_ctx_t ctx, int64_t m, int64_t n, int64_t d, const double* Y, int64_t ldy,
                     const double* T, int y_on_device, const double* h_history, double eps_r,
                     rbd_model_t* out) {
  if (!ctx || !out) return set_err(RBD_ERR_INVALID_ARGUMENT, "model_create: null context/output");
  if (m < 1 || n < 1 || d < 1 || d > n || ldy < m || !Y)
    return set_err(RBD_ERR_DIMENSION_MISMATCH, "model_create: inconsistent model shapes");
  CU(cudaSetDevice(ctx->device));
  auto* md = new rbd_model_s();
  md->device = ctx->device;
  md->m = m;
  md->n = n;
  md->d = d;
  md->eps_r = eps_r;
  if (h_history) md->history.assign(h_history, h_history + d);
  const cudaMemcpyKind kind = y_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  int rc = ensure(md->Y, sizeof(double) * (size_t)m * (size_t)d);
  if (rc == RBD_OK && T) rc = ensure(md->T, sizeof(double) * (size_t)d * (size_t)n);
  if (rc == RBD_OK &&
      (cudaMemcpy2DAsync(md->Y.p, sizeof(double) * m, Y, sizeof(double) * ldy, sizeof(double) * m,
                         d, kind, ctx->stream) != cudaSuccess ||
       (T && cudaMemcpyAsync(md->T.p, T, sizeof(double) * (size_t)d * (size_t)n, kind,
                             ctx->stream) != cudaSuccess) ||
       cudaStreamSynchronize(ctx->stream) != cudaSuccess))
    rc = set_err(RBD_ERR_CUDA, "model_create: copy failed");
  if (rc != RBD_OK) {
    rbd_model_free(md);
    return rc;
  }
  *out = md;
  return RBD_OK;
}

int rbd_model_load(rbd_ctx_t ctx, const char* path, rbd_model_t* out) {
  if (!ctx || !out) return set_err(RBD_ERR_INVALID_ARGUMENT, "model_load: null context/output");
  int64_t m, n, d;
  int tag;
  TRY(rbd_model_read_header(path, &m, &n, &d, &tag));
  CU(cudaSetDevice(ctx->device));
  auto* md = new rbd_model_s();
  md->device = ctx->device;
  md->m = m;
  md->n = n;
  md->d = d;
  md->weight_kind = tag;
  md->history.resize((size_t)d);
  if (tag == RBD_WEIGHT_DIAGONAL) md->diag.resize((size_t)m);
  int rc = ensure(md->Y, sizeof(double) * (size_t)m * (size_t)d);
  if (rc == RBD_OK) rc = ensure(md->T, sizeof(double) * (size_t)d * (size_t)n);
  if (rc == RBD_OK)
    rc = rbd_model_read(ctx, path, ptr<double>(md->Y), m, ptr<double>(md->T), &md->eps_r,
                        md->history.data(), md->diag.empty() ? nullptr : md->diag.data());
  if (rc != RBD_OK) {
    rbd_model_free(md);
    return rc;
  }
  *out = md;
  return RBD_OK;
}

int rbd_model_free(rbd_model_t md) {
  if (!md) return RBD_OK;
  cudaSetDevice(md->device);
  release(md->Y);
  release(md->T);
  release(md->Y32);
  delete md;
  return RBD_OK;
}

int rbd_model_info(rbd_model_t md, int64_t* m, int64_t* n, int64_t* d, const double** dY,
                   const double** dT, double* eps_r, int* weight_kind) {
  if (!md) return set_err(RBD_ERR_INVALID_ARGUMENT, "null model");
  if (m) *m = md->m;
  if (n) *n = md->n;
  if (d) *d = md->d;
  if (dY) *dY = ptr<double>(md->Y);
  if (dT) *dT = ptr<double>(md->T);
  if (eps_r) *eps_r = md->eps_r;
  if (weight_kind) *weight_kind = md->weight_kind;
  return RBD_OK;
}

int rbd_model_read_vectors(rbd_model_t md, double* h_history, double* h_diag) {
  if (!md) return set_err(RBD_ERR_INVALID_ARGUMENT, "null model");
  if (h_history) {
    if (md->history.empty()) std::fill(h_history, h_history + md->d, 0.0);
    else std::copy(md->history.begin(), md->history.end(), h_history);
  }
  if (h_diag && !md->diag.empty()) std::copy(md->diag.begin(), md->diag.end(), h_diag);
  return RBD_OK;
}

int rbd_project_model(rbd_ctx_t ctx, rbd_model_t md, const double* hXn, int64_t N, int64_t ldx,
                      double* hTn, double* h_err) {
  const double* xs[1] = {hXn};
  double* ts[1] = {hTn};
  double* es[1] = {h_err};
  return project_stream<double, double>(ctx, md, 1, xs, N, ldx, ts, h_err ? es : nullptr, false);
}

int rbd_project_host_many(rbd_ctx_t ctx, rbd_model_t md, int64_t count, const double* const* hXn,
                          int64_t N, int64_t ldx, double* const* hTn, double* const* h_err) {
  return project_stream<double, double>(ctx, md, count, hXn, N, ldx, hTn, h_err, false);
}

int rbd_project_host_many_f32(rbd_ctx_t ctx, rbd_model_t md, int64_t count,
                              const float* const* hXn, int64_t N, int64_t ldx, float* const* hTn,
                              double* const* h_err) {
  return project_stream<float, float>(ctx, md, count, hXn, N, ldx, hTn, h_err, true);
}

int rbd_reconstruct_model(rbd_ctx_t ctx, rbd_model_t md, const double* hC, int64_t N, double* hV) {
  TRY(check_model(ctx, md));
  if (N < 0) return set_err(RBD_ERR_DIMENSION_MISMATCH, "reconstruct: bad sizes");
  if (N == 0) return RBD_OK;
  if (!hC || !hV) return set_err(RBD_ERR_INVALID_ARGUMENT, "reconstruct: null buffers");
  CU(cudaSetDevice(ctx->device));
  const int64_t m = md->m, d = md->d;
  TRY(ensure(ctx->pm_T[0], sizeof(double) * (size_t)d * (size_t)N));
  TRY(ensure(ctx->pm_X[0], sizeof(double) * (size_t)m * (size_t)N));
  CU(cudaMemcpyAsync(ctx->pm_T[0].p, hC, sizeof(double) * (size_t)d * (size_t)N,
                     cudaMemcpyHostToDevice, ctx->stream));
  TRY(rbd_reconstruct_batch(ctx, ptr<double>(md->Y), m, d, m, ptr<double>(ctx->pm_T[0]), N,
                            ptr<double>(ctx->pm_X[0])));
  CU(cudaMemcpyAsync(hV, ctx->pm_X[0].p, sizeof(double) * (size_t)m * (size_t)N,
                     cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return RBD_OK;
}

}  // extern "C"
