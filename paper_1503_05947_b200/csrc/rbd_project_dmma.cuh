// rbd_project_dmma.cuh — out-of-sample compression T_new = Y' X_new on the
// FP64 tensor cores (DMMA: mma.sync.aligned.m16n8k4.row.col.f64), the one
// dense contraction of the path (BASELINE north_star).
//
// CTA tile BM (basis rows l) x BN (new columns j), K = rows i of Y / X_new in
// steps of 16 through a 3-stage cp.async pipeline. Both operands are staged
// K-contiguous exactly as they sit in global memory (Y and X_new are
// column-major) in XOR-swizzled 16-double rows (no padding). 64 x 64 tiles,
// 2 x 2 warps of 32 x 32, fragments loaded per k4 sub-step so a thread needs
// < 128 registers and four CTAs (16 warps) share an SM: the DMMA issue latency
// is hidden by warps.
// CTAs of the first l-tile also accumulate ||x_j||^2 from the staged X_new
// tiles (no second pass over X_new for the error indicator).
#pragma once

#include <cuda_runtime.h>

namespace rbdk {

constexpr int kDmBK = 16;           // i per stage (row of 16 doubles, no padding)
#ifndef RBD_DM_STAGES
#define RBD_DM_STAGES 3
#endif
#ifndef RBD_DM_MINB
#define RBD_DM_MINB 4
#endif
constexpr int kDmStages = RBD_DM_STAGES;

template <int BM, int BN>
constexpr size_t dm_smem_bytes() {
  return sizeof(double) * (size_t)kDmStages * (BM + BN) * kDmBK;
}

// XOR swizzle of the 16-double rows: element (row, k) lives at
// row*16 + (k ^ 4*(row & 3) ^ 2*(row & 1)). Keeps 16-byte chunks intact
// (cp.async). K5 permutes k inside a stage (lane t of DMMA step q takes
// k = 4t + q), so a lane's four elements of a row are one 32-byte group and
// load as two 16-byte halves; the row-parity bit puts the two rows of an
// 8-lane phase on different halves, which keeps those loads conflict free.
__device__ __forceinline__ int dm_swz(int row, int k) {
  return row * kDmBK + (k ^ ((row & 3) << 2) ^ ((row & 1) << 1));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// One stage of a K-contiguous operand: ROWS tile rows (columns of Y or X_new),
// 16 consecutive i each (8 chunks of 16 B). `full` = no bounds checks needed.
template <int ROWS, int NTHREADS>
__device__ __forceinline__ void dm_load_tile(double* s, const double* __restrict__ g, long long ld,
                                             long long r0, long long rmax, long long i0,
                                             long long m, bool full) {
  static_assert((ROWS * 8) % NTHREADS == 0, "loader split");
#pragma unroll
  for (int q = 0; q < ROWS * 8 / NTHREADS; ++q) {
    const int c = threadIdx.x + q * NTHREADS;
    const int row = c >> 3, ch = c & 7;
    const long long r = r0 + row;
    const long long i = i0 + ch * 2;
    int bytes = 16;
    if (!full) bytes = (r < rmax && i < m) ? ((i + 1 < m) ? 16 : 8) : 0;
    const double* src = (bytes > 0) ? g + r * ld + i : g;
    cp_async16(s + dm_swz(row, ch * 2), src, bytes);
  }
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int MINB = RBD_DM_MINB>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, MINB)
    k_project_dmma(const double* __restrict__ Y, long long m, long long d, long long ldy,
                   const double* __restrict__ Xn, long long N, long long ldx,
                   double* __restrict__ Tn, double* __restrict__ xnorm2, long long kc,
                   double* __restrict__ Tws, double* __restrict__ xws) {
  // split-K: blockIdx.z takes rows [z*kc, min(m, (z+1)*kc)) of Y / X_new (kc a
  // multiple of 16); split 0 writes Tn / xnorm2, split z > 0 its workspace slice
  {
    const long long z = blockIdx.z;
    const long long kb = z * kc, ke = (kb + kc < m) ? kb + kc : m;
    if (z > 0) {
      Tn = Tws + (z - 1) * d * N;
      if (xnorm2) xnorm2 = xws + (z - 1) * N;
    }
    Y += kb;
    Xn += kb;
    m = ke - kb;
  }
  constexpr int NTHREADS = WARPS_M * WARPS_N * 32;
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;   // warp tile
  constexpr int MT = WM / 16, NT = WN / 8;               // mma tiles per warp
  extern __shared__ __align__(16) double dm_smem[];
  double* As = dm_smem;                                  // [stages][BM][16] swizzled
  double* Bs = dm_smem + kDmStages * BM * kDmBK;         // [stages][BN][16] swizzled
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  // blockIdx.x = l-tile (fastest): the d/BM CTAs sharing an X_new tile run
  // together, so X_new streams from DRAM once and is re-read from L2
  const long long l0 = (long long)blockIdx.x * BM;
  const long long j0 = (long long)blockIdx.y * BN;
  const bool do_norm = (xnorm2 != nullptr) && blockIdx.x == 0;
  const bool fullA = (l0 + BM <= d), fullB = (j0 + BN <= N);
  double acc[MT][NT][4];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.0;
  // ||x_j||^2 (l-tile 0 only): each half of a B row (8 stored doubles) of
  // column (tid % BN) in two chains, halves combined in order. With 2 threads
  // per B row every thread takes one half; with one, a thread takes both halves
  // (separate chains), so the sum has the same bits for either tile shape.
  static_assert(NTHREADS == 2 * BN || NTHREADS == BN, "one or two threads per B row");
  constexpr int kHalves = 2 * BN / NTHREADS;   // halves per thread
  double xa = 0.0, xb = 0.0, xa2 = 0.0, xb2 = 0.0;
  __shared__ double xn_half[BN];
  const long long nk = (m + kDmBK - 1) / kDmBK;
  auto load_stage = [&](int st, long long kt) {
    const long long i0 = kt * kDmBK;
    const bool kfull = i0 + kDmBK <= m;
    dm_load_tile<BM, NTHREADS>(As + st * BM * kDmBK, Y, ldy, l0, d, i0, m, fullA && kfull);
    dm_load_tile<BN, NTHREADS>(Bs + st * BN * kDmBK, Xn, ldx, j0, N, i0, m, fullB && kfull);
  };
#pragma unroll
  for (int st = 0; st < kDmStages - 1; ++st) {
    if (st < nk) load_stage(st, st);
    cp_async_commit();
  }
  // every fragment row has (row & 3) == (g & 3) and (row & 1) == (g & 1): with
  // k = 4t + q, elements q = 2h, 2h+1 of the lane's group are the 16 bytes at
  // row*16 + 4*(t ^ (g & 3)) + 2*(h ^ (g & 1)), in q order
  const int baseA = (wm * WM + g) * kDmBK, baseB = (wn * WN + g) * kDmBK;
  const int off0 = 4 * (t ^ (g & 3)) + 2 * (g & 1), off1 = 4 * (t ^ (g & 3)) + 2 * ((g & 1) ^ 1);
  for (long long kt = 0; kt < nk; ++kt) {
    cp_async_wait<kDmStages - 2>();
    __syncthreads();
    {
      const long long kn = kt + kDmStages - 1;
      if (kn < nk) load_stage((int)(kn % kDmStages), kn);
      cp_async_commit();
    }
    const int sc = (int)(kt % kDmStages);
    const double* A = As + sc * BM * kDmBK;
    const double* B = Bs + sc * BN * kDmBK;
#pragma unroll
    for (int h = 0; h < 2; ++h) {   // DMMA steps q = 2h and 2h + 1
      const int off = h ? off1 : off0;
      double2 a0[MT], a1[MT], bf[NT];
#pragma unroll
      for (int a = 0; a < MT; ++a) {
        a0[a] = *reinterpret_cast<const double2*>(A + baseA + (a * 16) * kDmBK + off);
        a1[a] = *reinterpret_cast<const double2*>(A + baseA + (a * 16 + 8) * kDmBK + off);
      }
#pragma unroll
      for (int b = 0; b < NT; ++b)
        bf[b] = *reinterpret_cast<const double2*>(B + baseB + (b * 8) * kDmBK + off);
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b) dmma_16x8x4(acc[a][b], a0[a].x, a1[a].x, bf[b].x);
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b) dmma_16x8x4(acc[a][b], a0[a].y, a1[a].y, bf[b].y);
    }
    if (do_norm) {
      // stored positions p = 2q + h (the row's half h), rotated by the row so the
      // lanes of a warp spread over 8 bank pairs instead of one (rows are 128 B)
      const int row = tid % BN, h = (kHalves == 1) ? tid / BN : 0;
      const double* xr = B + row * kDmBK;
#pragma unroll
      for (int q = 0; q < kDmBK / 2; q += 2) {
        const double v0 = xr[(2 * q + h + 2 * row) & (kDmBK - 1)];
        const double v1 = xr[(2 * q + 2 + h + 2 * row) & (kDmBK - 1)];
        xa = fma(v0, v0, xa);
        xb = fma(v1, v1, xb);
        if (kHalves == 2) {
          const double u0 = xr[(2 * q + 1 + 2 * row) & (kDmBK - 1)];
          const double u1 = xr[(2 * q + 3 + 2 * row) & (kDmBK - 1)];
          xa2 = fma(u0, u0, xa2);
          xb2 = fma(u1, u1, xb2);
        }
      }
    }
  }
  cp_async_wait<0>();
  // epilogue: T_new is d x N column-major (ld d)
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const long long l = l0 + wm * WM + a * 16 + g + (e >= 2 ? 8 : 0);
        const long long j = j0 + wn * WN + b * 8 + t * 2 + (e & 1);
        if (l < d && j < N) Tn[l + j * d] = acc[a][b][e];
      }
  if (do_norm) {
    if (kHalves == 2) {
      if (j0 + tid < N) xnorm2[j0 + tid] = (xa + xb) + (xa2 + xb2);
    } else {
      if (tid >= BN) xn_half[tid - BN] = xa + xb;
      __syncthreads();
      if (tid < BN && j0 + tid < N) xnorm2[j0 + tid] = (xa + xb) + xn_half[tid];
    }
  }
}

// Split-K combine: Tn += workspace slices (and ||x||^2), splits in order.
static __global__ void k_splitk_sum(double* __restrict__ Tn, const double* __restrict__ Tws,
                             long long dN, int nws, double* __restrict__ xn,
                             const double* __restrict__ xws, long long N) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < dN;
       e += (long long)gridDim.x * blockDim.x) {
    double v = Tn[e];
    for (int z = 0; z < nws; ++z) v += Tws[(long long)z * dN + e];
    Tn[e] = v;
    if (xn && e < N) {
      double x = xn[e];
      for (int z = 0; z < nws; ++z) x += xws[(long long)z * N + e];
      xn[e] = x;
    }
  }
}

// err_j = max(||x_j||^2 - ||t_j||^2, 0) from the fused ||x||^2 (one warp per column).
static __global__ void k_project_err_fused(const double* __restrict__ xnorm2, const double* __restrict__ Tn,
                                    long long d, long long N, double* __restrict__ err) {
  const long long j = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (j >= N) return;
  double tt = 0.0;
  for (long long k = lane; k < d; k += 32) tt = fma(Tn[k + j * d], Tn[k + j * d], tt);
  for (int off = 16; off > 0; off >>= 1) tt += __shfl_xor_sync(0xffffffffu, tt, off);
  if (lane == 0) {
    const double e = xnorm2[j] - tt;
    err[j] = e > 0.0 ? e : 0.0;
  }
}

}  // namespace rbdk
