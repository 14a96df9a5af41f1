// rbd_project_tc.cuh — fp32 out-of-sample compression (K6) on the 5th-gen
// tensor cores: T_new = Y' X_new with tcgen05.mma kind::tf32 and a 3xTF32
// split, accumulators in TMEM, operands staged by TMA (128-byte swizzle).
// BASELINE north_star: "tcgen05 for the fp32 mode"; SURVEY §8(a) a9 (K6).
//
// 3xTF32: x = hi + lo with hi = x (the MMA reads the top 19 bits of the fp32
// container, i.e. truncates to tf32) and lo = x - tf32(x) (exact in fp32).
// D += A_hi B_hi + A_hi B_lo + A_lo B_hi recovers ~fp32 accuracy; only the lo
// tiles are computed (by the converter warps, in shared memory).
//
// CTA: 12 warps. warp 0 = TMA producer, warp 1 = TMEM owner + MMA issuer,
// warps 2-9 = converters (lo tiles) and then the epilogue (tcgen05.ld of their
// TMEM lane quarter, warp_id % 4, one column half each), warps 10-13 = the
// ||x_j||^2 accumulation in fp64 (Eq. 3), in the CTAs of the first l-tile row
// only. Tile 128 (l) x 128 (j), K = 32 fp32 rows (one 128-byte swizzle row)
// per stage, 3 stages.
// Eight converter warps and the norms in warps of their own: ncu showed the
// converters, not the tensor pipe or shared memory, pacing a k-block (four
// warps doing the split AND the fp32->fp64 widening + DFMA chains stalled
// 6-13 cycles per issued instruction); off the converters' path the norms
// only have to finish within a k-block's tensor time.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rbdk {

constexpr int kTcBM = 128;
constexpr int kTcBN = 128;
constexpr int kTcBK = 32;            // fp32 per 128-byte row
constexpr int kTcStages = 3;
constexpr int kTcConvWarps = 8;
constexpr int kTcXnWarps = 4;
constexpr int kTcXnRows = kTcBN / (32 * kTcXnWarps);   // B rows per norm thread
constexpr int kTcThreads = 64 + 32 * kTcConvWarps + 32 * kTcXnWarps;   // 448
constexpr int kTcTileBytes = kTcBM * kTcBK * 4;   // 16 KiB (A and B tiles are both 128 x 32)
// smem per stage: A raw, A lo, B raw, B lo
constexpr int kTcStageBytes = 4 * kTcTileBytes;
constexpr size_t kTcSmem = (size_t)kTcStages * kTcStageBytes + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: traps after ~20 s instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  unsigned spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if ((++spins & 0x3fffu) == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) __trap();
    }
  }
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major operand, 128-byte swizzle: 8-row atoms of 1024 B (SBO), version 1.
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* smem, uint32_t byte_off) {
  const uint32_t addr = smem_u32(smem) + byte_off;
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);            // start address [0,14)
  d |= (uint64_t)(16 >> 4) << 16;                    // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                  // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                            // version (sm100)
  d |= (uint64_t)2 << 61;                            // SWIZZLE_128B
  return d;
}

// kind::tf32, D f32, A/B tf32, both K-major, M = 128, N = kTcBN.
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4)                      // c_format = F32
         | (2u << 7)                    // a_format = TF32
         | (2u << 10)                   // b_format = TF32
         | ((uint32_t)(N >> 3) << 17)   // n_dim
         | ((uint32_t)(M >> 4) << 24);  // m_dim
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ float tf32_lo(float x) {
  const float hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);   // tf32 truncation
  return x - hi;                                                        // exact in fp32
}

// Converter thread t (0..255) of a stage: row r = t % 128 of the A tile and of
// the B tile, 16-byte chunks 4h..4h+3 (h = t / 128) of the row's 128 bytes: lo
// tiles written beside the raw ones.
__device__ __forceinline__ void tc_convert_half_rows(const uint8_t* A, uint8_t* Alo, const uint8_t* B, uint8_t* Blo,
                                                     int r, int h) {
  const float4* ar = reinterpret_cast<const float4*>(A + r * 128);
  float4* alo = reinterpret_cast<float4*>(Alo + r * 128);
  const float4* br = reinterpret_cast<const float4*>(B + r * 128);
  float4* blo = reinterpret_cast<float4*>(Blo + r * 128);
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    // same chunk position in raw and lo tiles; rotated per lane so the 8
    // lanes of a 128-byte phase hit 8 different bank groups
    const int c = (cc + 4 * h + r) & 7;
    const float4 a = ar[c];
    alo[c] = make_float4(tf32_lo(a.x), tf32_lo(a.y), tf32_lo(a.z), tf32_lo(a.w));
    const float4 b = br[c];
    blo[c] = make_float4(tf32_lo(b.x), tf32_lo(b.y), tf32_lo(b.z), tf32_lo(b.w));
  }
}

// ||x_j||^2 thread u of a stage: rows u + 32 kTcXnWarps rr of the raw B tile
// (columns j of X_new), each accumulated in four fp64 chains (the float4
// components) over the row's eight 16-byte chunks in rotated order.
__device__ __forceinline__ void tc_xnorm_rows(const uint8_t* B, int u, double (*xn)[4]) {
#pragma unroll
  for (int rr = 0; rr < kTcXnRows; ++rr) {
    const int r = u + 32 * kTcXnWarps * rr;
    const float4* br = reinterpret_cast<const float4*>(B + r * 128);
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const float4 b = br[(cc + r) & 7];
      xn[rr][0] = fma((double)b.x, (double)b.x, xn[rr][0]);
      xn[rr][1] = fma((double)b.y, (double)b.y, xn[rr][1]);
      xn[rr][2] = fma((double)b.z, (double)b.z, xn[rr][2]);
      xn[rr][3] = fma((double)b.w, (double)b.w, xn[rr][3]);
    }
  }
}

// split-K: blockIdx.z takes k-blocks [z * kb_per, min(nk, (z + 1) * kb_per)) (at
// least one); split 0 writes Tn / xnorm2, split z > 0 its workspace slices
// (Tws + (z-1) d N, xws + (z-1) N), added in order by k_splitk_sum_f32.
static __global__ void __launch_bounds__(kTcThreads, 1)
    k_project_tf32x3(const __grid_constant__ CUtensorMap mapY, const __grid_constant__ CUtensorMap mapX,
                     long long m, long long d, long long N, float* __restrict__ Tn,
                     double* __restrict__ xnorm2, int kb_per, float* __restrict__ Tws,
                     double* __restrict__ xws) {
  extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTcStages * kTcStageBytes);
  uint64_t* conv = full + kTcStages;
  uint64_t* empty = conv + kTcStages;
  uint64_t* tmem_full = empty + kTcStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int l0 = blockIdx.x * kTcBM, j0 = blockIdx.y * kTcBN;
  const int nk_all = (int)((m + kTcBK - 1) / kTcBK);
  const int kb0 = (int)blockIdx.z * kb_per;
  const int nk = (kb0 + kb_per < nk_all ? kb0 + kb_per : nk_all) - kb0;   // local k-blocks (>= 1)
  if (blockIdx.z > 0) {
    Tn = Tws + (long long)(blockIdx.z - 1) * d * N;
    if (xnorm2) xnorm2 = xws + (long long)(blockIdx.z - 1) * N;
  }

  const bool want_xn = xnorm2 != nullptr && blockIdx.x == 0;   // one l-tile row computes ||x_j||^2
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], kTcConvWarps);   // one arrival per converter warp
      mbar_init(&empty[s], want_xn ? 1 + kTcXnWarps : 1);   // MMA commit (+ the norm warps)
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {   // TMEM: kTcBN fp32 columns for the 128 x kTcBN accumulator
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTcBN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  auto stageA = [&](int s) { return smem + s * kTcStageBytes; };
  auto stageAlo = [&](int s) { return smem + s * kTcStageBytes + kTcTileBytes; };
  auto stageB = [&](int s) { return smem + s * kTcStageBytes + 2 * kTcTileBytes; };
  auto stageBlo = [&](int s) { return smem + s * kTcStageBytes + 3 * kTcTileBytes; };

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kTcStages;
        const uint32_t ph = (kb / kTcStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], 2 * kTcTileBytes);
        tma_load_2d(stageA(s), &mapY, &full[s], (kb0 + kb) * kTcBK, l0);
        tma_load_2d(stageB(s), &mapX, &full[s], (kb0 + kb) * kTcBK, j0);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_tf32(kTcBM, kTcBN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kTcStages;
        const uint32_t ph = (kb / kTcStages) & 1;
        // hi x hi needs only the TMA data; the two lo products wait for the
        // converters (they run while the first four MMAs execute)
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int kk = 0; kk < kTcBK / 8; ++kk) {   // K = 8 tf32 = 32 bytes per MMA
          const uint32_t off = kk * 32;
          umma_tf32(tmem, umma_desc_sw128(stageA(s), off), umma_desc_sw128(stageB(s), off), idesc,
                    (kb | kk) ? 1u : 0u);
        }
        mbar_wait(&conv[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int kk = 0; kk < kTcBK / 8; ++kk) {
          const uint32_t off = kk * 32;
          const uint64_t ah = umma_desc_sw128(stageA(s), off), al = umma_desc_sw128(stageAlo(s), off);
          const uint64_t bh = umma_desc_sw128(stageB(s), off), bl = umma_desc_sw128(stageBlo(s), off);
          umma_tf32(tmem, ah, bl, idesc, 1u);
          umma_tf32(tmem, al, bh, idesc, 1u);
        }
        umma_commit(&empty[s]);   // frees the stage once these MMAs complete
      }
      umma_commit(tmem_full);
    }
  } else if (warp >= 2 + kTcConvWarps) {
    // ---------------- ||x_j||^2 in fp64 (warps 10-13, first l-tile row only) ----------------
    if (want_xn) {
      const int u = threadIdx.x - 32 * (2 + kTcConvWarps);   // norm thread
      double xn[kTcXnRows][4] = {};
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kTcStages;
        const uint32_t ph = (kb / kTcStages) & 1;
        mbar_wait(&full[s], ph);
        tc_xnorm_rows(stageB(s), u, xn);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);   // this warp is done with the stage's raw B tile
      }
#pragma unroll
      for (int rr = 0; rr < kTcXnRows; ++rr)
        if (j0 + u + 32 * kTcXnWarps * rr < N) xnorm2[j0 + u + 32 * kTcXnWarps * rr] = (xn[rr][0] + xn[rr][1]) + (xn[rr][2] + xn[rr][3]);
    }
  } else {
    // ---------------- converters (warps 2-9): lo tiles ----------------
    const int t = threadIdx.x - 64;   // 0..255
    const int r = t & 127, h = t >> 7;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kTcStages;
      const uint32_t ph = (kb / kTcStages) & 1;
      mbar_wait(&full[s], ph);
      tc_convert_half_rows(stageA(s), stageAlo(s), stageB(s), stageBlo(s), r, h);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic -> async proxy
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[s]);
    }
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---------------- epilogue: TMEM -> registers -> T_new ----------------
    const int q = warp & 3;                 // TMEM lane quarter of this warp
    const int row = q * 32 + lane;          // accumulator row = basis index l0 + row
    const long long l = l0 + row;
#pragma unroll 1
    for (int c0 = h * (kTcBN / 2); c0 < (h + 1) * (kTcBN / 2); c0 += 32) {   // this warp's column half
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
          "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
            "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
            "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
            "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (l < d) {
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const long long j = j0 + c0 + c;
          if (j < N) Tn[l + j * d] = __uint_as_float(v[c]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcBN));
  }
}

// Split-K combine: Tn += fp32 workspace slices and xn += fp64 slices, in split order.
static __global__ void k_splitk_sum_f32(float* __restrict__ Tn, const float* __restrict__ Tws, long long dN,
                                 int nws, double* __restrict__ xn, const double* __restrict__ xws,
                                 long long N) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < dN;
       e += (long long)gridDim.x * blockDim.x) {
    float v = Tn[e];
    for (int z = 0; z < nws; ++z) v += Tws[(long long)z * dN + e];
    Tn[e] = v;
    if (xn && e < N) {
      double x = xn[e];
      for (int z = 0; z < nws; ++z) x += xws[(long long)z * N + e];
      xn[e] = x;
    }
  }
}

// err_j = max(||x_j||^2 - ||t_j||^2, 0), fp64 accumulation (the subtraction cancels).
static __global__ void k_project_err_f32(const double* __restrict__ xnorm2, const float* __restrict__ Tn,
                                  long long d, long long N, double* __restrict__ err) {
  const long long j = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (j >= N) return;
  double tt = 0.0;
  for (long long k = lane; k < d; k += 32) {
    const double t = Tn[k + j * d];
    tt = fma(t, t, tt);
  }
  for (int off = 16; off > 0; off >>= 1) tt += __shfl_xor_sync(0xffffffffu, tt, off);
  if (lane == 0) {
    const double e = xnorm2[j] - tt;
    err[j] = e > 0.0 ? e : 0.0;
  }
}

}  // namespace rbdk
