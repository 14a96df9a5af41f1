// rbd_project_tc2.cuh — K6 on a CTA pair: T_new = Y' X_new (fp32, 3xTF32) with
// tcgen05.mma.cta_group::2, one 256 (l) x 256 (j) tile per two-SM cluster.
//
// Why a pair: per 32-row k-block the single-CTA kernel (rbd_project_tc.cuh,
// 128 x 128 tile) moves 192 KB through shared memory (TMA writes 32 KB, the
// lo-tile converters read and write 64 KB, the twelve 128x128x8 MMAs read 8 KB
// of operands each) for 768 clk of tensor work at 128 B/clk. With
// cta_group::2 each CTA supplies its 128 rows of A (Y) and only HALF of B (128
// of the 256 X_new columns), and a 256x256x8 MMA takes 128 clk per SM: the
// same 192 KB per k-block feeds 1536 clk of tensor work. ncu on the C4 batch
// (profiles/r02k6f_*): shared-memory pipe 60 % -> 34 % of peak, tensor pipe
// 57 % -> 72 % of active cycles, 5.64 -> 4.78 ms with the error indicator.
// (A 4-deep raw ring + 2-deep lo ring in the same 192 KB measured the same:
// at this tensor load the clocks sit under the power cap.)
//
// Per CTA (rank r of the pair): A rows l0p + 128 r .. +127 (raw + lo tiles),
// B rows j0p + 128 r .. +127 (raw + lo), accumulator rows 128 r .. of D in its
// own TMEM (256 fp32 columns). Warp 0 = TMA producer (own tiles -> own `full`
// barrier), warps 2-9 = converters (lo tiles; each warp arrives once per stage
// on the LEADER's `conv` barrier, 16 arrivals), warps 10-13 = ||x_j||^2 in fp64
// for the CTA's own X_new columns (first l-tile row only), warp 1 of the
// leader issues the MMAs for the pair and commits with a 2-CTA multicast to
// both CTAs' `empty` / `tmem_full` barriers. Epilogue as in the single-CTA
// kernel, per CTA. Split-K and its in-order combine are shared with it.
// Same 3xTF32 arithmetic and fp32 accumulation chains per (l, j) as the
// single-CTA kernel at equal split-K (k-blocks in order), so the two agree
// bit for bit (tests/test_gpu_project_f32.py).
#pragma once

#include "rbd_project_tc.cuh"

namespace rbdk {

constexpr int kTc2BN = 256;          // pair tile: 256 (l) x 256 (j)
constexpr int kTc2Cols = 256;        // TMEM columns per CTA
constexpr int kTc2Stages = 3;
constexpr size_t kTc2Smem = (size_t)kTc2Stages * kTcStageBytes + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` (a shared::cta address of this CTA) in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(uint32_t p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(p), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait_cluster(bar, parity)) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  unsigned spins = 0;
  while (!mbar_try_wait_cluster(bar, parity)) {
    if ((++spins & 0x3fffu) == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) __trap();
    }
  }
}

__device__ __forceinline__ void umma2_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrives (once the pair's MMAs issued so far complete) on the barrier at this
// shared-memory offset in BOTH CTAs of the pair
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// grid (2 * ceil(d / 256), ceil(N / 256), splits), clusters of 2 along x.
static __global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTcThreads, 1)
    k_project_tf32x3_pair(const __grid_constant__ CUtensorMap mapY, const __grid_constant__ CUtensorMap mapX,
                          long long m, long long d, long long N, float* __restrict__ Tn,
                          double* __restrict__ xnorm2, int kb_per, float* __restrict__ Tws,
                          double* __restrict__ xws) {
  extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTc2Stages * kTcStageBytes);
  uint64_t* conv = full + kTc2Stages;      // used in the leader only (256 arrivals)
  uint64_t* empty = conv + kTc2Stages;
  uint64_t* tmem_full = empty + kTc2Stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int l0 = (int)(blockIdx.x >> 1) * 2 * kTcBM + (int)rank * kTcBM;   // this CTA's 128 rows of A / D
  const int j0p = (int)blockIdx.y * kTc2BN;                                // the pair's 256 columns
  const int jh = j0p + (int)rank * kTcBN;                                  // this CTA's half of B
  const int nk_all = (int)((m + kTcBK - 1) / kTcBK);
  const int kb0 = (int)blockIdx.z * kb_per;
  const int nk = (kb0 + kb_per < nk_all ? kb0 + kb_per : nk_all) - kb0;   // local k-blocks (>= 1)
  if (blockIdx.z > 0) {
    Tn = Tws + (long long)(blockIdx.z - 1) * d * N;
    if (xnorm2) xnorm2 = xws + (long long)(blockIdx.z - 1) * N;
  }

  const bool want_xn = xnorm2 != nullptr && (blockIdx.x >> 1) == 0;   // one l-tile row computes ||x_j||^2
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTc2Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 2 * kTcConvWarps);   // one arrival per converter warp of the pair
      mbar_init(&empty[s], want_xn ? 1 + kTcXnWarps : 1);   // the pair's MMA commit (+ own norm warps)
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();   // both CTAs' barriers exist before any remote arrive / multicast commit
  if (warp == 1) {      // TMEM: 256 fp32 columns in each CTA of the pair (same address in both)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTc2Cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  auto stageA = [&](int s) { return smem + s * kTcStageBytes; };
  auto stageAlo = [&](int s) { return smem + s * kTcStageBytes + kTcTileBytes; };
  auto stageB = [&](int s) { return smem + s * kTcStageBytes + 2 * kTcTileBytes; };
  auto stageBlo = [&](int s) { return smem + s * kTcStageBytes + 3 * kTcTileBytes; };

  if (warp == 0) {
    // ---------------- TMA producer (own tiles, own barriers) ----------------
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kTc2Stages;
        const uint32_t ph = (kb / kTc2Stages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], 2 * kTcTileBytes);
        tma_load_2d(stageA(s), &mapY, &full[s], (kb0 + kb) * kTcBK, l0);
        tma_load_2d(stageB(s), &mapX, &full[s], (kb0 + kb) * kTcBK, jh);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the leader CTA, for the pair ----------------
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = umma_idesc_tf32(2 * kTcBM, kTc2BN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kTc2Stages;
        const uint32_t ph = (kb / kTc2Stages) & 1;
        // 256 converter arrivals: both CTAs' raw tiles have landed and their lo tiles are written
        mbar_wait_cluster(&conv[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int kk = 0; kk < kTcBK / 8; ++kk) {   // K = 8 tf32 = 32 bytes per MMA; same order of
          const uint32_t off = kk * 32;            // products per k-block as the single-CTA kernel
          umma2_tf32(tmem, umma_desc_sw128(stageA(s), off), umma_desc_sw128(stageB(s), off), idesc,
                     (kb | kk) ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < kTcBK / 8; ++kk) {
          const uint32_t off = kk * 32;
          const uint64_t ah = umma_desc_sw128(stageA(s), off), al = umma_desc_sw128(stageAlo(s), off);
          const uint64_t bh = umma_desc_sw128(stageB(s), off), bl = umma_desc_sw128(stageBlo(s), off);
          umma2_tf32(tmem, ah, bl, idesc, 1u);
          umma2_tf32(tmem, al, bh, idesc, 1u);
        }
        umma2_commit_both(&empty[s]);   // frees the stage in both CTAs once these MMAs complete
      }
      umma2_commit_both(tmem_full);
    }
  } else if (warp >= 2 + kTcConvWarps) {
    // ---------------- ||x_j||^2 in fp64 (warps 10-13, first l-tile row only) ----------------
    if (want_xn) {
      const int u = threadIdx.x - 32 * (2 + kTcConvWarps);   // norm thread
      double xn[kTcXnRows][4] = {};
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kTc2Stages;
        const uint32_t ph = (kb / kTc2Stages) & 1;
        mbar_wait(&full[s], ph);
        tc_xnorm_rows(stageB(s), u, xn);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);   // this warp is done with the stage's raw B tile
      }
#pragma unroll
      for (int rr = 0; rr < kTcXnRows; ++rr)
        if (jh + u + 32 * kTcXnWarps * rr < N) xnorm2[jh + u + 32 * kTcXnWarps * rr] = (xn[rr][0] + xn[rr][1]) + (xn[rr][2] + xn[rr][3]);
    }
  } else {
    // ---------------- converters (warps 2-9): lo tiles ----------------
    const int t = threadIdx.x - 64;   // 0..255
    const int r = t & 127, h = t >> 7;
    const uint32_t conv_leader = mapa_u32(smem_u32(&conv[0]), 0);       // the leader's barriers
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kTc2Stages;
      const uint32_t ph = (kb / kTc2Stages) & 1;
      mbar_wait(&full[s], ph);
      tc_convert_half_rows(stageA(s), stageAlo(s), stageB(s), stageBlo(s), r, h);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic -> async proxy
      __syncwarp();
      // one cluster-scope release per warp (per thread it stalled the converters on the fence)
      if (lane == 0) mbar_arrive_cluster(conv_leader + (uint32_t)s * 8u);
    }
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---------------- epilogue: own TMEM (128 rows x 256 columns) -> T_new ----------------
    const int q = warp & 3;                 // TMEM lane quarter of this warp
    const int row = q * 32 + lane;          // accumulator row = basis index l0 + row
    const long long l = l0 + row;
#pragma unroll 1
    for (int c0 = h * (kTc2BN / 2); c0 < (h + 1) * (kTc2BN / 2); c0 += 32) {   // this warp's column half
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
          const long long j = j0p + c0 + c;
          if (j < N) Tn[l + j * d] = __uint_as_float(v[c]);
        }
      }
    }
  }
  // teardown: neither CTA may exit (or free TMEM) while the pair's MMAs, the
  // peer's remote arrives or the multicast commits can still touch it
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTc2Cols));
  }
}

}  // namespace rbdk
