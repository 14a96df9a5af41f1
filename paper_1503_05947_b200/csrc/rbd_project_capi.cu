// rbd_project_capi.cu — out-of-sample compression (K5 fp64 DMMA, K6 fp32
// tcgen05), reconstruct / compress_matrix, batched classify and the standalone
// sweep timer behind the C ABI (decompose.cpp:113-125, classify.cpp:22-34).
#include "rbd_capi_internal.h"
#include "rbd_project.cuh"
#include "rbd_project_tc.cuh"
#include "rbd_project_tc2.cuh"
#include "rbd_classify.cuh"
#include "rbd_compress_dmma.cuh"
#include "rbd_project_dmma_tma.cuh"

namespace {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D fp64 column-major operand for K5-TMA: rows (the K dimension, length
// `inner`) contiguous, `outer` columns of leading dimension ld; box 16 x 64,
// 128-byte swizzle (one 16-double row per 128 bytes).
int make_map_f64(CUtensorMap* map, const double* base, long long inner, long long outer, long long ld) {
  auto enc = tensor_map_encoder();
  if (!enc) return set_err(RBD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)rbdk::kDmBK, 64u};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(RBD_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return RBD_OK;
}

// K5 staging: 0 = per-thread cp.async (k_project_dmma), 1 = TMA, 3 stages, 4
// CTAs per SM (128 registers), 2 = TMA, 4 stages, 3 CTAs per SM (162
// registers, no spill). Measured on a C4 batch (tools/ab_k5.py, with the error
// indicator): 34.63 / 32.57 / 31.82 ms; ncu of mode 2: DMMA pipe active 97.3 %
// of active cycles (cuBLAS DGEMM, same operands: 30.41 ms). RBD_K5_TMA overrides.
int k5_tma_mode() {
  const char* e = getenv("RBD_K5_TMA");
  return e ? atoi(e) : 2;
}

// T_new (and ||x_j||^2) through k_project_dmma_tma; the caller combines
// split-K slices and forms the error indicator as for the cp.async kernel.
int launch_project_tma(rbd_ctx_t ctx, int mode, const double* dY, long long m, long long d, long long ldy,
                       const double* dXn, long long N, long long ldx, double* dTn, double* xn, int sk,
                       double* Tws, double* xws) {
  CUtensorMap mY, mX;
  TRY(make_map_f64(&mY, dY, m, d, ldy));
  TRY(make_map_f64(&mX, dXn, m, N, ldx));
  const long long kc = ((m + sk - 1) / sk + 15) / 16 * 16;
  dim3 grid((unsigned)cdiv(d, 64), (unsigned)cdiv(N, 64), (unsigned)sk);
  if (mode == 2) {
    static bool attr = false;
    if (!attr) {
      CU(cudaFuncSetAttribute(rbdk::k_project_dmma_tma<4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)rbdk::dt_smem_bytes<4>()));
      attr = true;
    }
    rbdk::k_project_dmma_tma<4, 3><<<grid, 128, rbdk::dt_smem_bytes<4>(), ctx->stream>>>(
        mY, mX, m, d, N, dTn, xn, kc, Tws, xws);
  } else {
    static bool attr = false;
    if (!attr) {
      CU(cudaFuncSetAttribute(rbdk::k_project_dmma_tma<3, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)rbdk::dt_smem_bytes<3>()));
      attr = true;
    }
    rbdk::k_project_dmma_tma<3, 4><<<grid, 128, rbdk::dt_smem_bytes<3>(), ctx->stream>>>(
        mY, mX, m, d, N, dTn, xn, kc, Tws, xws);
  }
  ctx->launches++;
  CU(cudaGetLastError());
  return RBD_OK;
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------------------
// Out-of-sample compression (K5) and reconstruct
// ---------------------------------------------------------------------------
int rbd_project_batch(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                      const double* dXn, int64_t N, int64_t ldx, double* dTn, double* d_err) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || N < 0) return set_err(RBD_ERR_DIMENSION_MISMATCH, "project: bad sizes");
  if (ldy < m || ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "project: vector length != m");
  if (N == 0) return RBD_OK;
  CU(cudaSetDevice(ctx->device));
  long long nl = 0;
  if (d_err) TRY(ensure(ctx->scratch1, sizeof(double) * (size_t)std::max<int64_t>(N, 32)));
  // split the K = m reduction when the DMMA grid would leave a partial last wave
  const int tma = k5_tma_mode();
  int sk = rbdk::project_splitk(m, d, N, ctx->nsm, tma == 2 ? 3 : (tma == 1 ? 4 : 0));
  if (sk > 1 && ensure(ctx->pj_ws, sizeof(double) * (size_t)(sk - 1) * (size_t)(d * N + N)) != RBD_OK)
    sk = 1;
  const bool tma_ok = tma > 0 && ldy % 2 == 0 && ldx % 2 == 0 && aligned16(dY) && aligned16(dXn) &&
                      m < (1LL << 31) && d < (1LL << 31) && N < (1LL << 31);
  if (tma_ok) {
    double* xn = d_err ? ptr<double>(ctx->scratch1) : nullptr;
    double* Tws = sk > 1 ? ptr<double>(ctx->pj_ws) : nullptr;
    double* xws = sk > 1 ? Tws + (long long)(sk - 1) * d * N : nullptr;
    TRY(launch_project_tma(ctx, tma, dY, m, d, ldy, dXn, N, ldx, dTn, xn, sk, Tws, xws));
    if (sk > 1) {
      rbdk::k_splitk_sum<<<1184, 256, 0, ctx->stream>>>(dTn, Tws, d * N, sk - 1, xn, xws, N);
      ctx->launches++;
    }
    if (d_err) {
      rbdk::k_project_err_fused<<<(unsigned)cdiv(N, 8), 256, 0, ctx->stream>>>(xn, dTn, d, N, d_err);
      ctx->launches++;
    }
    CU(cudaGetLastError());
    return RBD_OK;
  }
  int rc = rbdk::launch_project_f64(dY, m, d, ldy, dXn, N, ldx, dTn, d_err, ctx->stream, &nl,
                                    d_err ? ptr<double>(ctx->scratch1) : nullptr, sk,
                                    sk > 1 ? ptr<double>(ctx->pj_ws) : nullptr);
  ctx->launches += nl;
  if (rc != 0) return set_err(RBD_ERR_CUDA, std::string("project kernel: ") + cudaGetErrorString((cudaError_t)rc));
  return RBD_OK;
}

int rbd_nearest_columns(rbd_ctx_t ctx, const double* dC, int64_t d, int64_t Q, int64_t ldc,
                        const double* dT, int64_t n_train, int64_t* d_best, double* d_dist) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (d < 1 || n_train < 1 || Q < 0 || ldc < d)
    return set_err(RBD_ERR_DIMENSION_MISMATCH, "nearest: bad sizes");
  if (Q == 0) return RBD_OK;
  if (!dC || !dT || !d_best) return set_err(RBD_ERR_INVALID_ARGUMENT, "nearest: null buffer");
  CU(cudaSetDevice(ctx->device));
  const long long gx = cdiv(Q, kNnTile);
  const long long tiles = cdiv(n_train, kNnTile);
  // split the training columns for the best-filled waves (resident CTAs per SM
  // from the occupancy API); a larger split must fill them by 2 points more
  static int nn_occ = 0;
  if (nn_occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nn_occ, k_nearest, kThreads, 0) != cudaSuccess ||
        nn_occ < 1)
      nn_occ = 1;
  }
  const long long slots = (long long)nn_occ * ctx->nsm;
  long long nsplit = 1, per = tiles * kNnTile;
  {
    double best_eff = 0.0;
    for (long long sp = 1; sp <= std::min<long long>(tiles, 16); ++sp) {
      const long long pr = cdiv(tiles, sp) * kNnTile;
      const long long ns = cdiv(n_train, pr);
      const long long c = gx * ns, waves = cdiv(c, slots);
      const double eff = (double)c / (double)(waves * slots);
      if (sp == 1 || eff > best_eff + 0.02) {
        best_eff = eff;
        nsplit = ns;
        per = pr;
      }
    }
  }
  if (gx > 0x7fffffffLL || nsplit > 65535)
    return set_err(RBD_ERR_INVALID_ARGUMENT, "nearest: problem too large for one launch");
  TRY(ensure(ctx->nn_part, sizeof(NnRec) * (size_t)nsplit * (size_t)Q));
  k_nearest<<<dim3((unsigned)gx, (unsigned)nsplit), kThreads, 0, ctx->stream>>>(
      dC, ldc, dT, n_train, d, Q, per, ptr<NnRec>(ctx->nn_part));
  const int gr = (int)std::max<long long>(1, std::min<long long>(cdiv(Q, 256), (long long)ctx->nsm * 4));
  k_nearest_reduce<<<gr, 256, 0, ctx->stream>>>(ptr<NnRec>(ctx->nn_part), Q, (int)nsplit,
                                                reinterpret_cast<long long*>(d_best),
                                                d_dist);
  ctx->launches += 2;
  CU(cudaGetLastError());
  return RBD_OK;
}

int rbd_classify_batch(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                       const double* dT, int64_t n_train, const double* dQ, int64_t Q,
                       int64_t ldq, int64_t* d_best, double* d_dist) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || n_train < 1 || Q < 0)
    return set_err(RBD_ERR_DIMENSION_MISMATCH, "classify: bad sizes");
  if (ldy < m || ldq < m)
    return set_err(RBD_ERR_DIMENSION_MISMATCH, "classify: test dimension != training dimension");
  if (Q == 0) return RBD_OK;
  CU(cudaSetDevice(ctx->device));
  TRY(ensure(ctx->nn_coords, sizeof(double) * (size_t)d * (size_t)Q));
  double* C = ptr<double>(ctx->nn_coords);
  TRY(rbd_project_batch(ctx, dY, m, d, ldy, dQ, Q, ldq, C, nullptr));   // c = Y'v (K5)
  return rbd_nearest_columns(ctx, C, d, Q, d, dT, n_train, d_best, d_dist);
}

int rbd_classify_host(rbd_ctx_t ctx, const double* hY, int64_t m, int64_t d, const double* hT,
                      int64_t n_train, const double* hQ, int64_t Q, int64_t* h_best,
                      double* h_dist) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || n_train < 1 || Q < 0)
    return set_err(RBD_ERR_DIMENSION_MISMATCH, "classify: bad sizes");
  if (Q == 0) return RBD_OK;
  CU(cudaSetDevice(ctx->device));
  DevBuf &bY = ctx->hs[0], &bT = ctx->hs[1], &bQ = ctx->hs[2], &bB = ctx->hs[3],
         &bD = ctx->hs[4];   // context scratch, kept between calls
  auto fin = [&](int rc) { return rc; };
  const long long ldm = (m % 2 == 0) ? m : m + 1;   // 16-byte aligned columns for K5
  int rc;
  if ((rc = ensure(bY, sizeof(double) * ldm * d)) || (rc = ensure(bT, sizeof(double) * d * n_train)) ||
      (rc = ensure(bQ, sizeof(double) * ldm * Q)) || (rc = ensure(bB, sizeof(int64_t) * Q)) ||
      (rc = ensure(bD, sizeof(double) * Q)))
    return fin(rc);
  if (cudaMemcpy2DAsync(bY.p, sizeof(double) * ldm, hY, sizeof(double) * m, sizeof(double) * m, d,
                        cudaMemcpyHostToDevice, ctx->stream) ||
      cudaMemcpyAsync(bT.p, hT, sizeof(double) * d * n_train, cudaMemcpyHostToDevice, ctx->stream) ||
      cudaMemcpy2DAsync(bQ.p, sizeof(double) * ldm, hQ, sizeof(double) * m, sizeof(double) * m, Q,
                        cudaMemcpyHostToDevice, ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "classify_host: H2D failed"));
  rc = rbd_classify_batch(ctx, ptr<double>(bY), m, d, ldm, ptr<double>(bT), n_train, ptr<double>(bQ),
                          Q, ldm, ptr<int64_t>(bB), ptr<double>(bD));
  if (rc) return fin(rc);
  if (cudaMemcpyAsync(h_best, bB.p, sizeof(int64_t) * Q, cudaMemcpyDeviceToHost, ctx->stream) ||
      (h_dist && cudaMemcpyAsync(h_dist, bD.p, sizeof(double) * Q, cudaMemcpyDeviceToHost,
                                 ctx->stream)) ||
      cudaStreamSynchronize(ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "classify_host: D2H failed"));
  return fin(RBD_OK);
}

int rbd_reconstruct(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                    const double* dc, double* dv) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (ldy < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "reconstruct: ldy < m");
  CU(cudaSetDevice(ctx->device));
  long long nl = 0;
  int rc = rbdk::launch_reconstruct_f64(dY, m, d, ldy, dc, dv, ctx->stream, &nl);
  ctx->launches += nl;
  if (rc != 0) return set_err(RBD_ERR_CUDA, std::string("reconstruct kernel: ") + cudaGetErrorString((cudaError_t)rc));
  return RBD_OK;
}

}  // extern "C"

extern "C" {

int rbd_project_host(rbd_ctx_t ctx, const double* hY, int64_t m, int64_t d, const double* hXn,
                     int64_t N, double* hTn, double* h_err) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || N < 0) return set_err(RBD_ERR_DIMENSION_MISMATCH, "project: bad sizes");
  if (N == 0) return RBD_OK;
  CU(cudaSetDevice(ctx->device));
  DevBuf &bY = ctx->hs[0], &bX = ctx->hs[1], &bT = ctx->hs[2], &bE = ctx->hs[3];   // kept
  auto fin = [&](int rc) { return rc; };
  int rc;
  if ((rc = ensure(bY, sizeof(double) * m * d)) || (rc = ensure(bX, sizeof(double) * m * N)) ||
      (rc = ensure(bT, sizeof(double) * d * N)) || (rc = ensure(bE, sizeof(double) * N)))
    return fin(rc);
  if (cudaMemcpyAsync(bY.p, hY, sizeof(double) * m * d, cudaMemcpyHostToDevice, ctx->stream) ||
      cudaMemcpyAsync(bX.p, hXn, sizeof(double) * m * N, cudaMemcpyHostToDevice, ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "project_host: H2D failed"));
  rc = rbd_project_batch(ctx, ptr<double>(bY), m, d, m, ptr<double>(bX), N, m, ptr<double>(bT),
                         h_err ? ptr<double>(bE) : nullptr);
  if (rc) return fin(rc);
  if (hTn && cudaMemcpyAsync(hTn, bT.p, sizeof(double) * d * N, cudaMemcpyDeviceToHost, ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "project_host: D2H failed"));
  if (h_err && cudaMemcpyAsync(h_err, bE.p, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "project_host: D2H failed"));
  if (cudaStreamSynchronize(ctx->stream)) return fin(set_err(RBD_ERR_CUDA, "project_host: sync failed"));
  return fin(RBD_OK);
}

int rbd_reconstruct_host(rbd_ctx_t ctx, const double* hY, int64_t m, int64_t d, const double* hc,
                         double* hv) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 0) return set_err(RBD_ERR_DIMENSION_MISMATCH, "reconstruct: bad sizes");
  CU(cudaSetDevice(ctx->device));
  DevBuf &bY = ctx->hs[0], &bc = ctx->hs[1], &bv = ctx->hs[2];   // kept between calls
  auto fin = [&](int rc) { return rc; };
  int rc;
  if ((rc = ensure(bY, sizeof(double) * m * std::max<int64_t>(d, 1))) ||
      (rc = ensure(bc, sizeof(double) * std::max<int64_t>(d, 1))) || (rc = ensure(bv, sizeof(double) * m)))
    return fin(rc);
  if (d > 0 && (cudaMemcpyAsync(bY.p, hY, sizeof(double) * m * d, cudaMemcpyHostToDevice, ctx->stream) ||
                cudaMemcpyAsync(bc.p, hc, sizeof(double) * d, cudaMemcpyHostToDevice, ctx->stream)))
    return fin(set_err(RBD_ERR_CUDA, "reconstruct_host: H2D failed"));
  rc = rbd_reconstruct(ctx, ptr<double>(bY), m, d, m, ptr<double>(bc), ptr<double>(bv));
  if (rc) return fin(rc);
  if (cudaMemcpyAsync(hv, bv.p, sizeof(double) * m, cudaMemcpyDeviceToHost, ctx->stream) ||
      cudaStreamSynchronize(ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "reconstruct_host: D2H failed"));
  return fin(RBD_OK);
}

int rbd_time_sweep(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx,
                   const double* dy, int reps, double* ms_per_launch) {
  if (!ctx || reps < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "time_sweep: bad arguments");
  CU(cudaSetDevice(ctx->device));
  TRY(ensure(ctx->partial, sizeof(double) * cdiv(m, kChunk) * n));
  const int vec = (ldx % 2 == 0 && aligned16(dX) && aligned16(dy)) ? 2 : 1;
  SweepArgs s{};
  s.A = dX;
  s.lda = ldx;
  s.m = m;
  s.ncols = n;
  s.v = dy;
  s.partial = ptr<double>(ctx->partial);
  s.pstride = n;
  s.gate = GATE_NONE;
  TRY(launch_sweep(ctx, s, vec, MODE_DOT, true, n));  // warm-up
  cudaEvent_t a, b;
  CU(cudaEventCreate(&a));
  CU(cudaEventCreate(&b));
  cudaEventRecord(a, ctx->stream);
  for (int r = 0; r < reps; ++r) {
    int rc = launch_sweep(ctx, s, vec, MODE_DOT, true, n);
    if (rc) {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      return rc;
    }
  }
  cudaEventRecord(b, ctx->stream);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (e != cudaSuccess) return set_err(RBD_ERR_CUDA, std::string("time_sweep: ") + cudaGetErrorString(e));
  *ms_per_launch = ms / reps;
  return RBD_OK;
}

}  // extern "C"

extern "C" {

int rbd_reconstruct_batch(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                          const double* dC, int64_t N, double* dV) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (ldy < m || m < 1 || N < 0) return set_err(RBD_ERR_DIMENSION_MISMATCH, "compress: bad sizes");
  if (N == 0) return RBD_OK;
  CU(cudaSetDevice(ctx->device));
  if (d >= 1 && launch_compress_dmma<true>(dY, m, d, ldy, dC, N, d, dV, m, ctx->stream)) {
    ctx->launches += cdiv(cdiv(N, 64), 65535);
    CU(cudaGetLastError());
    return RBD_OK;
  }
  const long long gx = std::min<long long>(cdiv(m, 256), 1024);
  for (long long j0 = 0; j0 < N; j0 += 65535) {
    const long long nb = std::min<long long>(65535, N - j0);
    k_reconstruct_batch<<<dim3((unsigned)gx, (unsigned)nb), 256, 0, ctx->stream>>>(
        dY, m, d, ldy, dC + j0 * d, nb, dV + j0 * m);
    ctx->launches++;
  }
  CU(cudaGetLastError());
  return RBD_OK;
}

int rbd_compress_device(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                        const double* dT, int64_t n, int64_t ldt, double* dV, int64_t ldv) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || n < 0 || ldy < m || ldt < n || ldv < m)
    return set_err(RBD_ERR_DIMENSION_MISMATCH, "compress: bad sizes");
  if (n == 0) return RBD_OK;
  CU(cudaSetDevice(ctx->device));
  if (launch_compress_dmma<false>(dY, m, d, ldy, dT, n, ldt, dV, ldv, ctx->stream)) {
    ctx->launches += cdiv(cdiv(n, 64), 65535);
    CU(cudaGetLastError());
    return RBD_OK;
  }
  // unaligned operands: transpose T into column-major coefficients, SIMT path
  DevBuf c;
  TRY(ensure(c, sizeof(double) * (size_t)d * (size_t)n));
  for (int64_t k = 0; k < d; ++k)   // row k of T -> element k of every column
    CU(cudaMemcpy2DAsync(ptr<double>(c) + k, sizeof(double) * d, dT + k * ldt, sizeof(double),
                         sizeof(double), n, cudaMemcpyDeviceToDevice, ctx->stream));
  int rc = RBD_OK;
  if (ldv == m) {
    rc = rbd_reconstruct_batch(ctx, dY, m, d, ldy, ptr<double>(c), n, dV);
  } else {
    rc = set_err(RBD_ERR_INVALID_ARGUMENT, "compress: unaligned operands need ldv == m");
  }
  cudaStreamSynchronize(ctx->stream);
  release(c);
  return rc;
}

int rbd_compress_host(rbd_ctx_t ctx, const double* hY, int64_t m, int64_t d, const double* hC,
                      int64_t N, double* hV) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || N < 1) return set_err(RBD_ERR_DIMENSION_MISMATCH, "compress: bad sizes");
  CU(cudaSetDevice(ctx->device));
  DevBuf &bY = ctx->hs[0], &bC = ctx->hs[1], &bV = ctx->hs[2];   // kept between calls
  auto fin = [&](int rc) { return rc; };
  int rc;
  if ((rc = ensure(bY, sizeof(double) * m * d)) || (rc = ensure(bC, sizeof(double) * d * N)) ||
      (rc = ensure(bV, sizeof(double) * m * N)))
    return fin(rc);
  if (cudaMemcpyAsync(bY.p, hY, sizeof(double) * m * d, cudaMemcpyHostToDevice, ctx->stream) ||
      cudaMemcpyAsync(bC.p, hC, sizeof(double) * d * N, cudaMemcpyHostToDevice, ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "compress_host: H2D failed"));
  rc = rbd_reconstruct_batch(ctx, ptr<double>(bY), m, d, m, ptr<double>(bC), N, ptr<double>(bV));
  if (rc) return fin(rc);
  if (cudaMemcpyAsync(hV, bV.p, sizeof(double) * m * N, cudaMemcpyDeviceToHost, ctx->stream) ||
      cudaStreamSynchronize(ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "compress_host: D2H failed"));
  return fin(RBD_OK);
}

}  // extern "C"

// ===========================================================================
// fp32 out-of-sample compression on tcgen05 (K6)
// ===========================================================================
namespace {

// 2-D fp32 column-major operand (rows = contiguous dim of length `inner`,
// `outer` columns, leading dimension ld), box 32 x 128, 128-byte swizzle.
int make_map_f32(CUtensorMap* map, const float* base, long long inner, long long outer, long long ld) {
  auto enc = tensor_map_encoder();
  if (!enc) return set_err(RBD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)kTcBK, (cuuint32_t)kTcBM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(RBD_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return RBD_OK;
}

}  // namespace

extern "C" {

int rbd_project_batch_f32(rbd_ctx_t ctx, const float* dY, int64_t m, int64_t d, int64_t ldy,
                          const float* dXn, int64_t N, int64_t ldx, float* dTn, double* d_err) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || N < 0) return set_err(RBD_ERR_DIMENSION_MISMATCH, "project: bad sizes");
  if (ldy < m || ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "project: vector length != m");
  if (N == 0) return RBD_OK;
  if ((ldy % 4) || (ldx % 4) || !aligned16(dY) || !aligned16(dXn))
    return set_err(RBD_ERR_INVALID_ARGUMENT,
                   "project f32: leading dimensions must be multiples of 4 floats and bases 16-byte aligned (TMA)");
  CU(cudaSetDevice(ctx->device));
  CUtensorMap mY, mX;
  TRY(make_map_f32(&mY, dY, m, d, ldy));
  TRY(make_map_f32(&mX, dXn, m, N, ldx));
  static bool attr = false;
  if (!attr) {
    CU(cudaFuncSetAttribute(k_project_tf32x3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem));
    CU(cudaFuncSetAttribute(k_project_tf32x3_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTc2Smem));
    attr = true;
  }
  // CTA-pair kernel (tcgen05 cta_group::2, 256 x 256 tile per two SMs) once both
  // tile sides are used beyond a single CTA's 128; RBD_K6_PAIR=0/1 overrides
  bool pair = d > kTcBM && N > kTcBN;
  if (const char* e = getenv("RBD_K6_PAIR")) pair = atoi(e) != 0;
  if (pair) {
    // a device (or partition) that cannot co-schedule a two-CTA cluster of this
    // kernel takes the single-CTA kernel instead
    static int pair_ok = -1;
    if (pair_ok < 0) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(2, 1, 1);
      cfg.blockDim = dim3(kTcThreads, 1, 1);
      cfg.dynamicSmemBytes = kTc2Smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nclusters = 0;
      const cudaError_t ce = cudaOccupancyMaxActiveClusters(&nclusters, k_project_tf32x3_pair, &cfg);
      if (ce != cudaSuccess) cudaGetLastError();
      pair_ok = (ce == cudaSuccess && nclusters > 0) ? 1 : 0;
    }
    pair = pair_ok == 1;
  }
  double* xn = nullptr;
  if (d_err) {
    TRY(ensure(ctx->scratch1, sizeof(double) * (size_t)std::max<int64_t>(N, 32)));
    xn = ptr<double>(ctx->scratch1);
  }
  // split-K over the k-blocks for the best-filled waves (1 CTA per SM): 2 for C4's 4 x 128 tiles
  const long long nk = cdiv(m, kTcBK);
  // (pair: units are clusters, nsm / 2 of them per wave)
  const long long ctas = pair ? cdiv(d, 2 * kTcBM) * cdiv(N, kTc2BN) : cdiv(d, kTcBM) * cdiv(N, kTcBN);
  const long long slots = pair ? std::max(ctx->nsm / 2, 1) : ctx->nsm;
  int sk = 1;
  {
    double best_eff = 0.0;
    for (int s = 1; s <= 4; ++s) {
      if (s > 1 && nk / s < 64) break;
      const long long c = ctas * s, waves = cdiv(c, slots);
      const double eff = (double)c / (double)(waves * slots);
      if (s == 1 || eff > best_eff + 0.02) {
        sk = s;
        best_eff = eff;
      }
    }
  }
  if (const char* e = getenv("RBD_K6_SPLITK")) sk = (int)std::min<long long>(std::max(atoi(e), 1), nk);
  const int kb_per = (int)cdiv(nk, sk);
  sk = (int)cdiv(nk, kb_per);   // every split gets at least one k-block
  float* Tws = nullptr;
  double* xws = nullptr;
  if (sk > 1) {
    const size_t tbytes = sizeof(float) * (size_t)(sk - 1) * (size_t)(d * N);
    TRY(ensure(ctx->pj_ws, tbytes + sizeof(double) * (size_t)(sk - 1) * (size_t)N + 16));
    Tws = ptr<float>(ctx->pj_ws);
    xws = reinterpret_cast<double*>(reinterpret_cast<char*>(ctx->pj_ws.p) + ((tbytes + 15) & ~(size_t)15));
  }
  if (pair) {
    dim3 grid((unsigned)(2 * cdiv(d, 2 * kTcBM)), (unsigned)cdiv(N, kTc2BN), (unsigned)sk);
    k_project_tf32x3_pair<<<grid, kTcThreads, kTc2Smem, ctx->stream>>>(mY, mX, m, d, N, dTn, xn, kb_per,
                                                                        Tws, xws);
  } else {
    dim3 grid((unsigned)cdiv(d, kTcBM), (unsigned)cdiv(N, kTcBN), (unsigned)sk);
    k_project_tf32x3<<<grid, kTcThreads, kTcSmem, ctx->stream>>>(mY, mX, m, d, N, dTn, xn, kb_per,
                                                                  Tws, xws);
  }
  ctx->launches++;
  CU(cudaGetLastError());
  if (sk > 1) {
    k_splitk_sum_f32<<<1184, 256, 0, ctx->stream>>>(dTn, Tws, d * N, sk - 1, xn, xws, N);
    ctx->launches++;
    CU(cudaGetLastError());
  }
  if (d_err) {
    k_project_err_f32<<<(unsigned)cdiv(N, 8), 256, 0, ctx->stream>>>(xn, dTn, d, N, d_err);
    ctx->launches++;
    CU(cudaGetLastError());
  }
  return RBD_OK;
}

}  // extern "C"
