// Per-SM throughput of the fp32 -> fp64 widening on sm_100a, as used by the
// fp32-storage sweep (every element is widened, then one DFMA):
//   mode 0: DFMA only (fp64 operands)
//   mode 1: F2F.F64.F32 + DFMA
//   mode 2: integer widening (exponent rebias + mantissa shift; normal floats
//           and zero handled, subnormals flushed by a select) + DFMA
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 f2f_rate.cu -o f2f_rate
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double widen_int(float f) {
  const unsigned b = __float_as_uint(f);
  const unsigned mag = b & 0x7fffffffu;
  unsigned hi = (mag >> 3) + (896u << 20);
  hi = (mag < 0x00800000u) ? 0u : hi;            // zero / subnormal -> 0 (test only)
  hi |= b & 0x80000000u;
  return __hiloint2double((int)hi, (int)(b << 29));
}

template <int MODE>
__global__ void k(const float* in, double* out, int iters) {
  float f[8];
  double w[8], acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    f[i] = in[threadIdx.x * 8 + i];
    w[i] = 1.0 + i * 1e-3;
    acc[i] = 0.0;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double x;
      if (MODE == 0) x = w[(i + 1) & 7];
      else if (MODE == 1) x = (double)f[i];
      else x = widen_int(f[i]);
      acc[i] = fma(x, w[i], acc[i]);
      f[i] = __uint_as_float(__float_as_uint(f[i]) ^ 1u);   // defeat hoisting
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 1.25) out[0] = s;
}

template <int MODE>
void run(const char* nm, float* in, double* out, int sms) {
  const int iters = 4096, blocks = sms * 4, threads = 256;
  k<MODE><<<blocks, threads>>>(in, out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(in, out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double elems = (double)iters * 8 * blocks * threads;
  printf("%-22s %.1f G elem/s  (%.1f per SM per ns)  %s\n", nm, elems / best / 1e6,
         elems / best / 1e6 / sms, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* in;
  double* out;
  cudaMalloc(&in, 4096 * sizeof(float));
  cudaMemset(in, 0x3f, 4096 * sizeof(float));
  cudaMalloc(&out, 8);
  run<0>("DFMA only", in, out, sms);
  run<1>("F2F.F64.F32 + DFMA", in, out, sms);
  run<2>("int widen + DFMA", in, out, sms);
  return 0;
}
