// HBM streaming microbenchmark for the sweep's data movement on sm_100a:
// persistent grid (2 CTAs x 256 threads per SM), a dynamic tile queue of
// 4 columns x 4096 rows, column dot products with a vector held in L2.
//   mode 0: register loads (16 x 16 B per thread per tile, one batch)
//   mode 1: TMA 1D bulk copies into a shared-memory ring (NST stages of 16 KB,
//           mbarrier per stage, refilled by thread 0 after a CTA barrier)
//   mode 2: per-thread cp.async (16 B) ring in shared memory, NST stages, no
//           CTA barrier in the stream
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 stream_ring.cu -o stream_ring
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kT = 256, kChunk = 4096, kCols = 4;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE, int NST, typename XT>
__global__ void __launch_bounds__(kT, 2) k_stream(const XT* __restrict__ X, long long m, long long n,
                                                  const double* __restrict__ v, double* out,
                                                  unsigned long long* ctr) {
  constexpr int XV = 16 / sizeof(XT);           // elements per 16 B
  constexpr int SR = kT * XV;                   // rows per stage
  constexpr int Q = kChunk / SR;                // stages per tile
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bar[NST];
  __shared__ long long tq[64];
  __shared__ long long sh_t;
  const int tid = threadIdx.x;
  const long long S = m / kChunk, G = n / kCols, total = S * G;
  double acc[kCols] = {0, 0, 0, 0};
  auto fma_stage = [&](const XT* x0, const XT* x1, const XT* x2, const XT* x3, long long row) {
    const XT* xs[4] = {x0, x1, x2, x3};
    const double* vr = v + row;
#pragma unroll
    for (int c = 0; c < kCols; ++c)
#pragma unroll
      for (int e = 0; e < XV; ++e) acc[c] = fma((double)xs[c][e], vr[e], acc[c]);
  };
  if (MODE == 3) {   // fp32-style 8-column tiles, two batches of (Q/2 row groups x 8 columns)
    const long long G8 = n / 8, total8 = S * G8;
    double acc8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    while (true) {
      if (tid == 0) sh_t = (long long)atomicAdd(ctr, 1ull);
      __syncthreads();
      const long long t = sh_t;
      __syncthreads();
      if (t >= total8) break;
      const long long s = t / G8, g = t % G8;
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        uint4 xr[Q / 2][8];
        double2 wv[Q / 2][XV / 2];
#pragma unroll
        for (int q = 0; q < Q / 2; ++q) {
          const long long row = s * kChunk + (b * Q / 2 + q) * SR + tid * XV;
#pragma unroll
          for (int h = 0; h < XV / 2; ++h) wv[q][h] = __ldcg(reinterpret_cast<const double2*>(v + row) + h);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            xr[q][c] = __ldcs(reinterpret_cast<const uint4*>(X + (g * 8 + c) * m + row));
        }
#pragma unroll
        for (int q = 0; q < Q / 2; ++q)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const XT* xs = reinterpret_cast<const XT*>(&xr[q][c]);
            const double* ws = reinterpret_cast<const double*>(&wv[q][0]);
#pragma unroll
            for (int e = 0; e < XV; ++e) acc8[c] = fma((double)xs[e], ws[e], acc8[c]);
          }
      }
      __syncthreads();
    }
    acc[0] = acc8[0] + acc8[1] + acc8[2] + acc8[3] + acc8[4] + acc8[5] + acc8[6] + acc8[7];
  } else if (MODE == 0) {
    while (true) {
      if (tid == 0) sh_t = (long long)atomicAdd(ctr, 1ull);
      __syncthreads();
      const long long t = sh_t;
      __syncthreads();
      if (t >= total) break;
      const long long s = t / G, g = t % G;
      uint4 xr[Q][kCols];
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int c = 0; c < kCols; ++c)
          xr[q][c] = __ldcs(reinterpret_cast<const uint4*>(X + (g * kCols + c) * m + s * kChunk + q * SR) + tid);
#pragma unroll
      for (int q = 0; q < Q; ++q)
        fma_stage(reinterpret_cast<const XT*>(&xr[q][0]), reinterpret_cast<const XT*>(&xr[q][1]),
                  reinterpret_cast<const XT*>(&xr[q][2]), reinterpret_cast<const XT*>(&xr[q][3]),
                  s * kChunk + q * SR + tid * XV);
    }
  } else {
    // claim queue ahead: tid 0 keeps the FIFO tq of tiles (claimed in order)
    // items = (tile, q); item i lives in slot i % NST
    long long nclaimed = 0;   // (tid 0)
    if (tid == 0) {
      for (int i = 0; i < NST; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      // claim enough tiles to cover NST stages + one
      for (int i = 0; i < (NST + Q - 1) / Q + 1; ++i) tq[nclaimed++ & 63] = (long long)atomicAdd(ctr, 1ull);
    }
    __syncthreads();
    long long item_iss = 0, item_cons = 0;   // uniform
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    auto issue = [&](long long it) {   // item it -> slot
      const long long t = tq[(it / Q) & 63];
      if (t >= total) return false;
      const int q = (int)(it % Q);
      const long long s = t / G, g = t % G;
      unsigned char* dst = smem + (it % NST) * (kCols * 4096);
      if (MODE == 1) {
        if (tid == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[it % NST])),
                       "r"(kCols * 4096) : "memory");
#pragma unroll
          for (int c = 0; c < kCols; ++c)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
                "%2, [%3], %4;" ::"r"(su32(dst + c * 4096)),
                "l"(X + (g * kCols + c) * m + s * kChunk + q * SR), "r"(4096), "r"(su32(&bar[it % NST])), "l"(pol)
                : "memory");
        }
      } else {
#pragma unroll
        for (int c = 0; c < kCols; ++c)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + c * 4096 + 16 * tid)),
                       "l"(X + (g * kCols + c) * m + s * kChunk + q * SR + tid * XV) : "memory");
      }
      return true;
    };
    // prologue
    for (int i = 0; i < NST; ++i) {
      issue(item_iss);
      ++item_iss;
      if (MODE == 2) asm volatile("cp.async.commit_group;" ::: "memory");
    }
    while (true) {
      const long long t = tq[(item_cons / Q) & 63];
      if (t >= total) break;
      const int q = (int)(item_cons % Q);
      const long long s = t / G;
      const unsigned slot = (unsigned)(item_cons % NST);
      if (MODE == 1) {
        const unsigned par = (unsigned)((item_cons / NST) & 1);
        unsigned ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(su32(&bar[slot])), "r"(par) : "memory");
      } else {
        asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1) : "memory");
      }
      const unsigned char* sp = smem + slot * (kCols * 4096) + 16 * tid;
      uint4 xr[kCols];
#pragma unroll
      for (int c = 0; c < kCols; ++c) xr[c] = *reinterpret_cast<const uint4*>(sp + c * 4096);
      ++item_cons;
      if (MODE == 1) __syncthreads();
      // tile boundary bookkeeping: claim one more tile when a new tile starts
      if (item_cons % Q == 0) {
        if (MODE == 2) __syncthreads();
        if (tid == 0) tq[nclaimed++ & 63] = (long long)atomicAdd(ctr, 1ull);
        __syncthreads();
      }
      issue(item_iss);
      ++item_iss;
      if (MODE == 2) asm volatile("cp.async.commit_group;" ::: "memory");
      fma_stage(reinterpret_cast<const XT*>(&xr[0]), reinterpret_cast<const XT*>(&xr[1]),
                reinterpret_cast<const XT*>(&xr[2]), reinterpret_cast<const XT*>(&xr[3]),
                s * kChunk + q * SR + tid * XV);
    }
    if (MODE == 2) asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  double sum = acc[0] + acc[1] + acc[2] + acc[3];
  if (sum == 1.2345) out[0] = sum;
}

template <int MODE, int NST, typename XT>
void run(const char* name, XT* X, long long m, long long n, double* v, double* out, unsigned long long* ctr,
         int sms) {
  const size_t smem = MODE == 0 ? 0 : (size_t)NST * kCols * 4096;
  cudaFuncSetAttribute(k_stream<MODE, NST, XT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stream<MODE, NST, XT>, kT, smem);
  const int grid = sms * (occ < 2 ? occ : 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaMemset(ctr, 0, 8);
    cudaEventRecord(e0);
    k_stream<MODE, NST, XT><<<grid, kT, smem>>>(X, m, n, v, out, ctr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;
  }
  const double bytes = (double)m * n * sizeof(XT);
  printf("%-28s elt=%zu grid=%d: %.3f ms  %.0f GB/s  (%s)\n", name, sizeof(XT), grid, best,
         bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  const int sel = argc > 1 ? atoi(argv[1]) : -1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long m = 32768, n = 2432 * 2;   // ~637 MB fp64
  double* Xd;
  float* Xf;
  double *v, *out;
  unsigned long long* ctr;
  cudaMalloc(&Xd, sizeof(double) * m * n);
  cudaMalloc(&Xf, sizeof(float) * m * n);
  cudaMalloc(&v, sizeof(double) * m);
  cudaMalloc(&out, 8);
  cudaMalloc(&ctr, 8);
  cudaMemset(Xd, 0, sizeof(double) * m * n);
  cudaMemset(Xf, 0, sizeof(float) * m * n);
  cudaMemset(v, 0, sizeof(double) * m);
  if (sel < 0 || sel == 10) run<3, 1, double>("regs 8col 2 batches", Xd, m, n, v, out, ctr, sms);
  if (sel < 0 || sel == 11) run<3, 1, float>("regs 8col 2 batches", Xf, m, n, v, out, ctr, sms);
  if (sel < 0 || sel == 0) run<0, 1, double>("regs", Xd, m, n, v, out, ctr, sms);
  if (sel < 0 || sel == 1) run<1, 4, double>("tma ring 4", Xd, m, n, v, out, ctr, sms);
  if (sel < 0 || sel == 2) run<1, 6, double>("tma ring 6", Xd, m, n, v, out, ctr, sms);
  if (sel < 0 || sel == 3) run<2, 4, double>("cp.async ring 4", Xd, m, n, v, out, ctr, sms);
  if (sel < 0 || sel == 4) run<2, 6, double>("cp.async ring 6", Xd, m, n, v, out, ctr, sms);
  if (sel < 0 || sel == 5) run<0, 1, float>("regs", Xf, m, n, v, out, ctr, sms);
  if (sel < 0 || sel == 6) run<1, 4, float>("tma ring 4", Xf, m, n, v, out, ctr, sms);
  if (sel < 0 || sel == 7) run<1, 6, float>("tma ring 6", Xf, m, n, v, out, ctr, sms);
  if (sel < 0 || sel == 8) run<2, 4, float>("cp.async ring 4", Xf, m, n, v, out, ctr, sms);
  if (sel < 0 || sel == 9) run<2, 6, float>("cp.async ring 6", Xf, m, n, v, out, ctr, sms);
  return 0;
}
