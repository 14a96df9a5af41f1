// Microbenchmark: can P1 read its Y row blocks in R-row segments (R x 8 bytes
// per column, stride m between columns) at HBM speed? That decides whether a
// P1 that keeps each block in shared memory (so Y'w1 needs no second HBM read
// of Y) is viable. Y: m x k fp64 column-major; every CTA takes a contiguous
// row range, processed in R-row blocks: all k columns of the block are copied
// into shared memory with cp.async (16 B per op), then consumed (w1 = x - Y c
// and p += Y'w1 on the block, from shared memory). NB buffers per CTA: with 2
// the copy of block b+1 overlaps the math of block b.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 p1_blocks.cu -o p1_blocks
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kT = 256;

__device__ __forceinline__ void cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)),
               "l"(g));
}

template <int R, int NB, bool COPY_ONLY>
__global__ void __launch_bounds__(kT) k_blocks(const double* __restrict__ Y, long long m, int k,
                                              const double* __restrict__ c, double* out) {
  extern __shared__ __align__(16) double sm[];   // [NB][k][R]
  __shared__ double w1[R];
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const long long lo = (m * cta / G) / R * R, hi = (cta + 1 == G) ? m : (m * (cta + 1) / G) / R * R;
  const int nblk = (int)((hi - lo) / R);
  double pacc = 0.0;   // thread-owned column tid (k <= 256 per thread slot, else strided)
  constexpr int CH = R / 2;   // 16-byte chunks per column segment
  auto issue = [&](int b) {
    if (b >= nblk) return;
    double* dst = sm + (size_t)(b % NB) * k * R;
    const long long r0 = lo + (long long)b * R;
    for (int e = tid; e < k * CH; e += kT) {
      const int col = e / CH, ch = e % CH;
      cp16(dst + col * R + ch * 2, Y + (long long)col * m + r0 + ch * 2);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  for (int b = 0; b < NB - 1; ++b) issue(b);
  for (int b = 0; b < nblk; ++b) {
    issue(b + NB - 1);
    if (NB == 2) asm volatile("cp.async.wait_group 1;\n" ::);
    else asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    const double* s = sm + (size_t)(b % NB) * k * R;
    if (COPY_ONLY) {   // the copy alone: one element per thread consumed
      pacc += s[tid % (k * R)];
      __syncthreads();
      continue;
    }
    // w1 rows: R rows, k columns (threads split rows x column slices)
    if (tid < R) {
      double acc = 0.0;
      for (int col = 0; col < k; ++col) acc = fma(s[col * R + tid], c[col], acc);
      w1[tid] = 1.0 - acc;
    }
    __syncthreads();
    for (int col = tid; col < k; col += kT) {
      double sum = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) sum = fma(s[col * R + r], w1[r], sum);
      pacc += sum;
    }
    __syncthreads();
  }
  if (pacc == 12345.0) out[cta] = pacc;   // keep the work
}

// Baseline: the P1 access pattern of the loop (lanes own row pairs of a 128-row
// block, columns split over the 4 warps of a half, 16 loads in flight per lane).
__global__ void __launch_bounds__(kT, 2) k_p1(const double* __restrict__ Y, long long m, int k,
                                             const double* __restrict__ c, double* out) {
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long lo = ((m * cta / G) + 1) & ~1LL, hi = (cta + 1 == G) ? m : (((m * (cta + 1) / G) + 1) & ~1LL);
  double acc = 0.0;
  for (long long rb = lo; rb < hi; rb += 128) {
    const int half = warp / 4, wh = warp % 4;
    const long long i0 = rb + half * 64 + 2 * lane;
    if (i0 + 1 >= hi) continue;
    const double* yp = Y + i0 + (long long)wh * m;
    for (int l = wh; l < k; l += 64) {
      double2 v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q)
        v[q] = (l + q * 4 < k) ? __ldcg(reinterpret_cast<const double2*>(yp + (long long)q * 4 * m))
                               : make_double2(0, 0);
#pragma unroll
      for (int q = 0; q < 16; ++q) acc = fma(v[q].x + v[q].y, c[(l + q * 4) & 511], acc);
      yp += 64 * m;
    }
  }
  if (acc == 12345.0) out[cta] = acc;
}

// P1 pattern with wider per-column segments: a lane owns RPL row pairs of a
// half (2*RPL rows), so each column segment of a block is 64*RPL*8*2 bytes;
// 16 loads in flight per lane (16/RPL columns per batch).
template <int RPL>
__global__ void __launch_bounds__(kT, 2) k_p1w(const double* __restrict__ Y, long long m, int k,
                                              const double* __restrict__ c, double* out) {
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int HR = 64 * RPL;          // rows per half
  constexpr int CB = 16 / RPL;          // columns per batch per warp
  const long long lo = ((m * cta / G) + 1) & ~1LL, hi = (cta + 1 == G) ? m : (((m * (cta + 1) / G) + 1) & ~1LL);
  double acc = 0.0;
  for (long long rb = lo; rb < hi; rb += 2 * HR) {
    const int half = warp / 4, wh = warp % 4;
    const long long i0 = rb + half * HR + 2 * lane;
    for (int l = wh; l < k; l += 4 * CB) {
      double2 v[CB][RPL];
#pragma unroll
      for (int q = 0; q < CB; ++q)
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const long long i = i0 + 64 * r;
          v[q][r] = (l + q * 4 < k && i + 1 < hi)
                        ? __ldcg(reinterpret_cast<const double2*>(Y + i + (long long)(l + q * 4) * m))
                        : make_double2(0, 0);
        }
#pragma unroll
      for (int q = 0; q < CB; ++q)
#pragma unroll
        for (int r = 0; r < RPL; ++r) acc = fma(v[q][r].x + v[q][r].y, c[(l + q * 4) & 511], acc);
    }
  }
  if (acc == 12345.0) out[cta] = acc;
}

int main(int argc, char** argv) {
  const long long m = argc > 1 ? atoll(argv[1]) : (1 << 20);
  const int k = argc > 2 ? atoi(argv[2]) : 512;
  double *Y, *c, *out;
  cudaMalloc(&Y, sizeof(double) * m * k);
  cudaMalloc(&c, sizeof(double) * 4096);
  cudaMalloc(&out, sizeof(double) * 4096);
  cudaMemset(Y, 0, sizeof(double) * m * k);
  cudaMemset(c, 0, sizeof(double) * 4096);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = (double)m * k * 8;
  auto timeit = [&](auto launch, const char* name) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    cudaError_t e = cudaGetLastError();
    printf("%-34s %8.3f ms  %7.1f GB/s  %s\n", name, best, bytes / best / 1e6,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  timeit([&] { k_p1<<<2 * nsm, kT>>>(Y, m, k, c, out); }, "P1 pattern (128-row blocks, regs)");
  timeit([&] { k_p1w<1><<<2 * nsm, kT>>>(Y, m, k, c, out); }, "P1 RPL=1 (1 KB segments)");
  timeit([&] { k_p1w<2><<<2 * nsm, kT>>>(Y, m, k, c, out); }, "P1 RPL=2 (2 KB segments)");
  timeit([&] { k_p1w<4><<<2 * nsm, kT>>>(Y, m, k, c, out); }, "P1 RPL=4 (4 KB segments)");
  timeit([&] { k_p1w<8><<<2 * nsm, kT>>>(Y, m, k, c, out); }, "P1 RPL=8 (8 KB segments)");
#define RUN(R, NB, CPS, CO)                                                                \
  {                                                                                        \
    const size_t smb = sizeof(double) * (size_t)NB * k * R;                                \
    if (smb * CPS <= 220 * 1024) {                                                         \
      cudaFuncSetAttribute(k_blocks<R, NB, CO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb); \
      char nm[64];                                                                         \
      snprintf(nm, sizeof nm, "smem R=%d NB=%d %d CTA/SM%s", R, NB, CPS, CO ? " copy" : "");   \
      timeit([&] { k_blocks<R, NB, CO><<<CPS * nsm, kT, smb>>>(Y, m, k, c, out); }, nm);   \
    }                                                                                      \
  }
  RUN(8, 2, 2, true);
  RUN(16, 2, 1, true);
  RUN(16, 1, 2, true);
  RUN(32, 1, 1, true);
  RUN(8, 4, 1, true);
  RUN(16, 2, 1, false);
  return 0;
}
