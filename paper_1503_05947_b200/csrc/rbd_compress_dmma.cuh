// rbd_compress_dmma.cuh — compress_matrix / reconstruct batch V = Y B on the
// FP64 tensor cores (reference decompose.cpp:119-125:
// reconstruct = Y c, compress_matrix = Y T).
//
// V (m x N, column-major, ld ldv) = Y (m x d, column-major, ld ldy) * B (d x N),
// with B either the decompose T as the library stores it (row-major,
// B(k, j) = T[k*ldb + j]) or a column-major coefficient block (B(k, j) =
// C[j*ldb + k]). K = d is small (<= a few thousand), M = m and N large.
// CTA tile 64 (i) x 64 (j), 2 x 2 warps of 32 x 32, K in steps of 16 through a
// 3-stage cp.async pipeline (same DMMA m16n8k4 core as K5). Y (M-contiguous)
// and a row-major T (N-contiguous) are staged as 16 K-rows of 64 + 4 doubles:
// the padding makes the fragment loads (k = 4q + t, row g / g + 8)
// conflict-free; a column-major B reuses K5's swizzled K-contiguous stage.
#pragma once

#include "rbd_project_dmma.cuh"

namespace rbdk {

constexpr int kGcPad = 4;

template <int BM, int BN, bool BKC>
constexpr size_t gc_smem_bytes() {
  return sizeof(double) * (size_t)kDmStages *
         ((size_t)kDmBK * (BM + kGcPad) + (BKC ? (size_t)BN * kDmBK : (size_t)kDmBK * (BN + kGcPad)));
}

// One stage of an operand that is contiguous along the tile's long axis:
// 16 K-rows (k0 .. k0+15) of COLS contiguous doubles starting at column c0,
// element (kk, cc) = g[(k0 + kk) * ld + c0 + cc], stored at s[kk*(COLS+pad) + cc].
template <int COLS, int NTHREADS>
__device__ __forceinline__ void gc_load_rows(double* s, const double* __restrict__ g, long long ld,
                                             long long c0, long long cmax, long long k0,
                                             long long kmax, bool full) {
  constexpr int CH = COLS / 2;   // 16-byte chunks per K-row
  static_assert((kDmBK * CH) % NTHREADS == 0, "loader split");
#pragma unroll
  for (int q = 0; q < kDmBK * CH / NTHREADS; ++q) {
    const int c = threadIdx.x + q * NTHREADS;
    const int kk = c / CH, ch = c % CH;
    const long long k = k0 + kk, col = c0 + ch * 2;
    int bytes = 16;
    if (!full) bytes = (k < kmax && col < cmax) ? ((col + 1 < cmax) ? 16 : 8) : 0;
    const double* src = (bytes > 0) ? g + k * ld + col : g;
    cp_async16(s + kk * (COLS + kGcPad) + ch * 2, src, bytes);
  }
}

template <int BM, int BN, int WARPS_M, int WARPS_N, bool BKC>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, 4)
    k_compress_dmma(const double* __restrict__ Y, long long m, long long d, long long ldy,
                    const double* __restrict__ Bm, long long N, long long ldb,
                    double* __restrict__ V, long long ldv) {
  constexpr int NTHREADS = WARPS_M * WARPS_N * 32;
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  constexpr int MT = WM / 16, NT = WN / 8;
  constexpr int SA = kDmBK * (BM + kGcPad);                      // doubles per A stage
  constexpr int SB = BKC ? BN * kDmBK : kDmBK * (BN + kGcPad);   // doubles per B stage
  extern __shared__ __align__(16) double gc_smem[];
  double* As = gc_smem;
  double* Bs = gc_smem + kDmStages * SA;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  const long long i0 = (long long)blockIdx.x * BM;   // rows of V (fastest: CTAs share a B tile)
  const long long j0 = (long long)blockIdx.y * BN;
  const bool fullA = i0 + BM <= m, fullB = j0 + BN <= N;
  double acc[MT][NT][4];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.0;
  const long long nk = (d + kDmBK - 1) / kDmBK;
  auto load_stage = [&](int st, long long kt) {
    const long long k0 = kt * kDmBK;
    const bool kfull = k0 + kDmBK <= d;
    gc_load_rows<BM, NTHREADS>(As + st * SA, Y, ldy, i0, m, k0, d, fullA && kfull);
    if constexpr (BKC)
      dm_load_tile<BN, NTHREADS>(Bs + st * SB, Bm, ldb, j0, N, k0, d, fullB && kfull);
    else
      gc_load_rows<BN, NTHREADS>(Bs + st * SB, Bm, ldb, j0, N, k0, d, fullB && kfull);
  };
#pragma unroll
  for (int st = 0; st < kDmStages - 1; ++st) {
    if (st < nk) load_stage(st, st);
    cp_async_commit();
  }
  int koff[4];   // swizzled K-contiguous B stage (BKC, dm_swz): (row, 4q + t)
#pragma unroll
  for (int q = 0; q < 4; ++q) koff[q] = 4 * (q ^ (g & 3)) + (t ^ ((g & 1) << 1));
  const int rowA = wm * WM + g, colB = wn * WN + g;
  for (long long kt = 0; kt < nk; ++kt) {
    cp_async_wait<kDmStages - 2>();
    __syncthreads();
    {
      const long long kn = kt + kDmStages - 1;
      if (kn < nk) load_stage((int)(kn % kDmStages), kn);
      cp_async_commit();
    }
    const int sc = (int)(kt % kDmStages);
    const double* A = As + sc * SA;
    const double* B = Bs + sc * SB;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int kk = 4 * q + t;
      double af[MT][2], bf[NT];
#pragma unroll
      for (int a = 0; a < MT; ++a) {
        af[a][0] = A[kk * (BM + kGcPad) + rowA + a * 16];
        af[a][1] = A[kk * (BM + kGcPad) + rowA + a * 16 + 8];
      }
#pragma unroll
      for (int b = 0; b < NT; ++b)
        bf[b] = BKC ? B[(colB + b * 8) * kDmBK + koff[q]] : B[kk * (BN + kGcPad) + colB + b * 8];
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b) dmma_16x8x4(acc[a][b], af[a][0], af[a][1], bf[b]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const long long i = i0 + wm * WM + a * 16 + g + (e >= 2 ? 8 : 0);
        const long long j = j0 + wn * WN + b * 8 + t * 2 + (e & 1);
        if (i < m && j < N) V[i + j * ldv] = acc[a][b][e];
      }
}

// V = Y B; false when the DMMA path's alignment needs are not met (ld even,
// 16-byte aligned bases), in which case the caller uses the SIMT kernel.
template <bool BKC>
inline bool launch_compress_dmma(const double* Y, long long m, long long d, long long ldy,
                                 const double* Bm, long long N, long long ldb, double* V,
                                 long long ldv, cudaStream_t s) {
  if ((ldy % 2) || (ldb % 2) ||
      ((reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(Bm)) & 15))
    return false;
  constexpr int BM = 64, BN = 64;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_compress_dmma<BM, BN, 2, 2, BKC>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)gc_smem_bytes<BM, BN, BKC>());
    attr = true;
  }
  const long long gx = (m + BM - 1) / BM, gy = (N + BN - 1) / BN;
  for (long long y0 = 0; y0 < gy; y0 += 65535) {   // grid.y limit
    const long long ny = (gy - y0 < 65535) ? gy - y0 : 65535;
    const long long jofs = y0 * BN;
    k_compress_dmma<BM, BN, 2, 2, BKC><<<dim3((unsigned)gx, (unsigned)ny), 128,
                                         gc_smem_bytes<BM, BN, BKC>(), s>>>(
        Y, m, d, ldy, BKC ? Bm + jofs * ldb : Bm + jofs, N - jofs, ldb, V + jofs * ldv, ldv);
  }
  return true;
}

}  // namespace rbdk
