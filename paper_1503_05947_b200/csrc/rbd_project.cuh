// rbd_project.cuh — out-of-sample compression T_new = Y' X_new with the
// identity error indicator err_j = max(||x_j||^2 - ||t_j||^2, 0)
// (reference: project decompose.cpp:113-117 per vector; Eq.(3) PAPER.md:273-279,
// workspace.cpp:88-97), and reconstruct v = Y c (decompose.cpp:119-123).
//
// fp64 tile kernel on the FP64 pipe: 64x64 output tile per CTA, K-step 16,
// double-buffered shared-memory staging, 4x4 register micro-tile per thread.
#pragma once

#include <cuda_runtime.h>

#include "rbd_project_dmma.cuh"

namespace rbdk {

constexpr int kPjBM = 64;   // rows of T_new (basis index k) per CTA
constexpr int kPjBN = 64;   // columns of T_new (new vectors) per CTA
constexpr int kPjBK = 16;   // reduction depth per stage (rows i of Y / X_new)

static __global__ void __launch_bounds__(256) k_project_f64(const double* __restrict__ Y, long long m,
                                                     long long d, long long ldy,
                                                     const double* __restrict__ Xn, long long N,
                                                     long long ldx, double* __restrict__ Tn) {
  __shared__ double As[2][kPjBK][kPjBM + 2];
  __shared__ double Bs[2][kPjBK][kPjBN + 2];
  const int t = threadIdx.x;
  const int tx = t % 16, ty = t / 16;
  const long long k0 = (long long)blockIdx.y * kPjBM;
  const long long j0 = (long long)blockIdx.x * kPjBN;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  const int li = t % 16, lc = t / 16;  // loader: row-in-stage, column group
  auto load = [&](int buf, long long i0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int col = lc + 16 * q;
      const long long i = i0 + li;
      const long long kk = k0 + col, jj = j0 + col;
      As[buf][li][col] = (i < m && kk < d) ? Y[i + kk * ldy] : 0.0;
      Bs[buf][li][col] = (i < m && jj < N) ? Xn[i + jj * ldx] : 0.0;
    }
  };
  load(0, 0);
  __syncthreads();
  int buf = 0;
  for (long long i0 = 0; i0 < m; i0 += kPjBK) {
    if (i0 + kPjBK < m) load(buf ^ 1, i0 + kPjBK);
#pragma unroll
    for (int ii = 0; ii < kPjBK; ++ii) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[buf][ii][ty * 4 + a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[buf][ii][tx * 4 + b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const long long kk = k0 + ty * 4 + a, jj = j0 + tx * 4 + b;
      if (kk < d && jj < N) Tn[kk + jj * d] = acc[a][b];
    }
}

// err_j = max(||x_j||^2 - ||t_j||^2, 0), one warp per column (fixed order).
static __global__ void k_project_err(const double* __restrict__ Xn, long long m, long long ldx,
                              const double* __restrict__ Tn, long long d, long long N,
                              double* __restrict__ err) {
  const long long j = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (j >= N) return;
  const double* x = Xn + j * ldx;
  double xx = 0.0, tt = 0.0;
  for (long long i = lane; i < m; i += 32) xx = fma(x[i], x[i], xx);
  for (long long k = lane; k < d; k += 32) tt = fma(Tn[k + j * d], Tn[k + j * d], tt);
  for (int off = 16; off > 0; off >>= 1) {
    xx += __shfl_xor_sync(0xffffffffu, xx, off);
    tt += __shfl_xor_sync(0xffffffffu, tt, off);
  }
  if (lane == 0) {
    const double e = xx - tt;
    err[j] = e > 0.0 ? e : 0.0;
  }
}

static __global__ void k_reconstruct(const double* __restrict__ Y, long long m, long long d,
                              long long ldy, const double* __restrict__ c, double* __restrict__ v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (long long k = 0; k < d; ++k) s = fma(Y[i + k * ldy], c[k], s);
    v[i] = s;
  }
}

// Split-K factor for the DMMA grid (4 CTAs per SM): of 1..4 (>= 1024 rows per
// split), the one whose waves are best filled; a larger split must fill them
// by 2 points more (its combine pass and workspace are not free). E.g. C4's
// 8 x 256 tiles -> 2 (6.92 waves), classify's 7 x 256 -> 4 (12.1 waves, 93 %
// instead of 3.03 waves at 76 %).
// K5 tile shape: 0 = 64 x 64 CTA tiles of 2 x 2 warps (32 x 32 each), 4 CTAs
// per SM; 1 = 64 x 128 tiles of 2 x 2 warps (32 x 64 each: twice the DMMAs per
// fragment load and per CTA barrier), 2 CTAs per SM. RBD_K5_TILE overrides.
inline int project_tile() {
  const char* e = getenv("RBD_K5_TILE");
  return e ? atoi(e) : 0;
}

inline int project_splitk(long long m, long long d, long long N, int nsm, int per_sm = 0) {
  const int tile = project_tile();
  const long long bn = tile == 1 ? 128 : 64;
  const long long ctas = ((d + 63) / 64) * ((N + bn - 1) / bn);
  const long long slots = (per_sm > 0 ? per_sm : (tile == 1 ? 2LL : 4LL)) * nsm;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 4; ++s) {
    if (s > 1 && m / s < 1024) break;
    const long long c = ctas * s;
    const long long waves = (c + slots - 1) / slots;
    const double eff = (double)c / (double)(waves * slots);
    if (s == 1 || eff > best_eff + 0.02) {
      best = s;
      best_eff = eff;
    }
  }
  return best;
}

inline int launch_project_f64(const double* Y, long long m, long long d, long long ldy,
                              const double* Xn, long long N, long long ldx, double* Tn,
                              double* err, cudaStream_t s, long long* nlaunch,
                              double* xnorm_scratch = nullptr, int splitk = 1,
                              double* splitk_ws = nullptr) {
  const bool dmma_ok = (ldy % 2 == 0) && (ldx % 2 == 0) &&
                       ((reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(Xn)) & 15) == 0;
  *nlaunch = 0;
  if (dmma_ok) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_project_dmma<64, 64, 2, 2>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm_smem_bytes<64, 64>());
      cudaFuncSetAttribute(k_project_dmma<64, 128, 2, 2, 2>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dm_smem_bytes<64, 128>());
      attr = true;
    }
    double* xn = err ? xnorm_scratch : nullptr;
    const int sk = (splitk > 1 && splitk_ws) ? splitk : 1;
    // workspace layout: (sk-1) T slices of d*N, then (sk-1) ||x||^2 slices of N
    double* Tws = splitk_ws;
    double* xws = splitk_ws ? splitk_ws + (long long)(sk - 1) * d * N : nullptr;
    const long long kc = ((m + sk - 1) / sk + 15) / 16 * 16;
    if (project_tile() == 1) {
      dim3 grid((unsigned)((d + 63) / 64), (unsigned)((N + 127) / 128), (unsigned)sk);
      k_project_dmma<64, 128, 2, 2, 2><<<grid, 128, dm_smem_bytes<64, 128>(), s>>>(
          Y, m, d, ldy, Xn, N, ldx, Tn, xn, kc, Tws, xws);
    } else {
      dim3 grid((unsigned)((d + 63) / 64), (unsigned)((N + 63) / 64), (unsigned)sk);
      k_project_dmma<64, 64, 2, 2><<<grid, 128, dm_smem_bytes<64, 64>(), s>>>(
          Y, m, d, ldy, Xn, N, ldx, Tn, xn, kc, Tws, xws);
    }
    *nlaunch += 1;
    if (sk > 1) {
      k_splitk_sum<<<1184, 256, 0, s>>>(Tn, Tws, d * N, sk - 1, xn, xws, N);
      *nlaunch += 1;
    }
    if (err) {
      k_project_err_fused<<<(unsigned)((N + 7) / 8), 256, 0, s>>>(xn, Tn, d, N, err);
      *nlaunch += 1;
    }
    return (int)cudaGetLastError();
  }
  dim3 grid((unsigned)((N + kPjBN - 1) / kPjBN), (unsigned)((d + kPjBM - 1) / kPjBM));
  k_project_f64<<<grid, 256, 0, s>>>(Y, m, d, ldy, Xn, N, ldx, Tn);
  *nlaunch = 1;
  if (err) {
    k_project_err<<<(unsigned)((N + 7) / 8), 256, 0, s>>>(Xn, m, ldx, Tn, d, N, err);
    *nlaunch += 1;
  }
  return (int)cudaGetLastError();
}

// V = Y C (decompose.cpp:119-125): thread per row i, one column j per grid.y.
static __global__ void k_reconstruct_batch(const double* __restrict__ Y, long long m, long long d,
                                    long long ldy, const double* __restrict__ C, long long N,
                                    double* __restrict__ V) {
  const long long j = blockIdx.y;
  const double* c = C + j * d;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (long long k = 0; k < d; ++k) s = fma(Y[i + k * ldy], c[k], s);
    V[i + j * m] = s;
  }
}

inline int launch_reconstruct_f64(const double* Y, long long m, long long d, long long ldy,
                                  const double* c, double* v, cudaStream_t s, long long* nlaunch) {
  const long long g = (m + 255) / 256;
  k_reconstruct<<<(unsigned)(g < 4096 ? g : 4096), 256, 0, s>>>(Y, m, d, ldy, c, v);
  *nlaunch = 1;
  return (int)cudaGetLastError();
}

}  // namespace rbdk
