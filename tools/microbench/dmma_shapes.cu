// DMMA issue-rate microbenchmark: m16n8k4 / m16n8k8 / m16n8k16 f64 on sm_100a.
// Each warp runs ACC independent accumulator chains for ITERS iterations with
// register-resident operands; reports TFLOP/s for the whole GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_shapes.cu -o dmma_shapes
#include <cstdio>
#include <cuda_runtime.h>

template <int K, int ACC>
__global__ void k_dmma(double* out, int iters, double seed) {
  double a[K / 2 > 1 ? K / 2 : 1][2], b[K / 4], c[ACC][4];
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < (K / 2 > 1 ? K / 2 : 1); ++i) { a[i][0] = seed * (lane + i); a[i][1] = seed - i; }
#pragma unroll
  for (int i = 0; i < K / 4; ++i) b[i] = seed + lane * i;
#pragma unroll
  for (int x = 0; x < ACC; ++x)
#pragma unroll
    for (int e = 0; e < 4; ++e) c[x][e] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int x = 0; x < ACC; ++x) {
      if constexpr (K == 4) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[x][0]), "+d"(c[x][1]), "+d"(c[x][2]), "+d"(c[x][3])
                     : "d"(a[0][0]), "d"(a[0][1]), "d"(b[0]));
      } else if constexpr (K == 8) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[x][0]), "+d"(c[x][1]), "+d"(c[x][2]), "+d"(c[x][3])
                     : "d"(a[0][0]), "d"(a[0][1]), "d"(a[1][0]), "d"(a[1][1]), "d"(b[0]), "d"(b[1]));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[x][0]), "+d"(c[x][1]), "+d"(c[x][2]), "+d"(c[x][3])
                     : "d"(a[0][0]), "d"(a[0][1]), "d"(a[1][0]), "d"(a[1][1]), "d"(a[2][0]), "d"(a[2][1]),
                       "d"(a[3][0]), "d"(a[3][1]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int x = 0; x < ACC; ++x) s += c[x][0] + c[x][1] + c[x][2] + c[x][3];
  if (s == 12345.678) out[0] = s;
}

template <int K, int ACC>
void run(int blocks_per_sm, int warps) {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 4096;
  dim3 grid(sms * blocks_per_sm), block(32 * warps);
  k_dmma<K, ACC><<<grid, block>>>(out, 16, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dmma<K, ACC><<<grid, block>>>(out, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 16 * 8 * K * (double)ACC * iters * grid.x * warps;
  printf("m16n8k%-2d acc=%d warps/blk=%d blk/SM=%d : %.2f TFLOP/s (%.3f ms) err=%s\n", K, ACC, warps,
         blocks_per_sm, flops / best * 1e-9, best, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<4, 8>(1, w);
    run<8, 8>(1, w);
    run<16, 8>(1, w);
  }
  run<4, 4>(2, 16);
  run<8, 4>(2, 16);
  run<16, 4>(2, 16);
  return 0;
}
