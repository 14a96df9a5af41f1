// rbd_project_dmma_tma.cuh — K5 with TMA staging: T_new = Y' X_new on the FP64
// tensor cores (DMMA m16n8k4), operands brought into shared memory by the
// tensor memory accelerator instead of per-thread cp.async.
//
// Same CTA tile as k_project_dmma (64 basis rows l x 64 new columns j, 2 x 2
// warps of 32 x 32, 4 CTAs per SM) and the same K order (k = 4t + q inside
// each 16-row stage, stages in order), so T_new has the same bits. What
// changes is the staging:
//  * one elected thread issues two cp.async.bulk.tensor.2d per stage (A = Y,
//    B = X_new, box 16 rows x 64 columns, 128-byte swizzle) that complete on
//    the stage's "full" mbarrier (expect_tx); no thread computes addresses;
//  * warps release a stage through its "empty" mbarrier (4 arrivals) instead
//    of a CTA barrier, so the four warps drift independently; the elected
//    thread refills a stage once all four warps are through it;
//  * out-of-range rows / columns (partial tiles, the tail of the last split)
//    are zero-filled by the TMA unit: no bounds checks in the loop.
// The 128-byte swizzle keeps the fragment loads conflict free: lane (g, t)
// reads logical 16-byte chunk 2t + h of tile row r (r & 7 == g), stored at
// chunk (2t + h) ^ g, so an 8-lane phase covers 8 distinct chunks.
// CTAs of l-tile 0 also accumulate ||x_j||^2 from the staged X_new tiles.
#pragma once

#include "rbd_project_dmma.cuh"
#include "rbd_project_tc.cuh"

namespace rbdk {

constexpr int kDtTile = 64 * kDmBK * 8;   // bytes of one operand stage (64 rows x 16 doubles)

template <int STAGES>
constexpr size_t dt_smem_bytes() {
  return (size_t)STAGES * 2 * kDtTile + 1024 /*align*/ + 2 * STAGES * 8 /*barriers*/ + 64 * 8;
}

template <int STAGES, int MINB>
__global__ void __launch_bounds__(128, MINB)
    k_project_dmma_tma(const __grid_constant__ CUtensorMap mY, const __grid_constant__ CUtensorMap mX,
                       long long m, long long d, long long N, double* __restrict__ Tn,
                       double* __restrict__ xnorm2, long long kc, double* __restrict__ Tws,
                       double* __restrict__ xws) {
  constexpr int BN = 64, WN = 32, WM = 32, MT = 2, NT = 4, WARPS_N = 2;
  extern __shared__ __align__(1024) uint8_t dt_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dt_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * 2 * kDtTile);
  uint64_t* empty = full + STAGES;
  double* xn_half = reinterpret_cast<double*>(empty + STAGES);
  // split-K: rows [kb, min(m, kb + kc)) of Y / X_new (kc a multiple of 16)
  const long long kb = (long long)blockIdx.z * kc;
  const long long ke = (kb + kc < m) ? kb + kc : m;
  if (blockIdx.z > 0) {
    Tn = Tws + (long long)(blockIdx.z - 1) * d * N;
    if (xnorm2) xnorm2 = xws + (long long)(blockIdx.z - 1) * N;
  }
  const long long nk = (ke - kb + kDmBK - 1) / kDmBK;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  const int l0 = (int)blockIdx.x * 64, j0 = (int)blockIdx.y * BN;
  const bool do_norm = (xnorm2 != nullptr) && blockIdx.x == 0;
  auto stA = [&](long long s) { return reinterpret_cast<const double*>(sm + s * 2 * kDtTile); };
  auto stB = [&](long long s) { return reinterpret_cast<const double*>(sm + s * 2 * kDtTile + kDtTile); };
  auto issue = [&](long long kt) {   // (elected thread) stage kt % STAGES <- k-tile kt
    const int s = (int)(kt % STAGES);
    mbar_expect_tx(&full[s], 2 * kDtTile);
    const int i0 = (int)(kb + kt * kDmBK);
    tma_load_2d(sm + s * 2 * kDtTile, &mY, &full[s], i0, l0);
    tma_load_2d(sm + s * 2 * kDtTile + kDtTile, &mX, &full[s], i0, j0);
  };
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (long long kt = 0; kt < STAGES && kt < nk; ++kt) issue(kt);
  }
  __syncthreads();

  double acc[MT][NT][4];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.0;
  double xa = 0.0, xb = 0.0;
  // fragment rows: A row wm*32 + a*16 + g (+8), B row wn*32 + b*8 + g; all have
  // (row & 7) == g, so chunk 2t + h sits at ((2t + h) ^ g) * 2 doubles
  const int baseA = (wm * WM + g) * kDmBK, baseB = (wn * WN + g) * kDmBK;
  const int off0 = 2 * ((2 * t) ^ g), off1 = 2 * ((2 * t + 1) ^ g);
  // ||x_j||^2: thread tid takes half hh of row r (logical chunks 4hh .. 4hh+3)
  const int nr = tid & 63, nh = tid >> 6;
  for (long long kt = 0; kt < nk; ++kt) {
    // refill the stage every warp released in iteration kt - 1
    if (tid == 0 && kt >= 1 && kt - 1 + STAGES < nk) {
      mbar_wait(&empty[(kt - 1) % STAGES], (uint32_t)(((kt - 1) / STAGES) & 1));
      issue(kt - 1 + STAGES);
    }
    const long long s = kt % STAGES;
    mbar_wait(&full[s], (uint32_t)((kt / STAGES) & 1));
    const double* A = stA(s);
    const double* B = stB(s);
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
      const double* xr = B + nr * kDmBK;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double2 v = *reinterpret_cast<const double2*>(xr + 2 * ((4 * nh + c) ^ (nr & 7)));
        xa = fma(v.x, v.x, xa);
        xb = fma(v.y, v.y, xb);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
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
    if (nh == 1) xn_half[nr] = xa + xb;
    __syncthreads();
    if (nh == 0 && j0 + nr < N) xnorm2[j0 + nr] = (xa + xb) + xn_half[nr];
  }
}

}  // namespace rbdk
