// Grid-barrier latency microbenchmark (cooperative launch, 2 CTAs/SM x 256 threads).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int VARIANT>
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = gen + 1;
    if (VARIANT == 0) {  // fence + atomic + sleep-spin (current)
      __threadfence();
      if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
        bar[0] = 0u;
        __threadfence();
        atomicAdd(&bar[1], 1u);
      } else {
        while (ld_acquire_u32(&bar[1]) != target) __nanosleep(64);
      }
      __threadfence();
    } else if (VARIANT == 1) {  // fence + atomic + pure spin
      __threadfence();
      if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
        bar[0] = 0u;
        __threadfence();
        atomicAdd(&bar[1], 1u);
      } else {
        while (ld_acquire_u32(&bar[1]) != target) {}
      }
      __threadfence();
    } else {  // release-add on a monotonic counter, acquire spin on it (no reset)
      unsigned old;
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
      const unsigned goal = (old / gridDim.x + 1) * gridDim.x;
      while (true) {
        unsigned v = ld_acquire_u32(bar);
        if ((int)(v - goal) >= 0) break;
      }
    }
    gen = target;
  }
  __syncthreads();
}

template <int VARIANT>
__global__ void __launch_bounds__(256, 2) k(unsigned* bar, int iters) {
  unsigned gen = 0;
  if (threadIdx.x == 0) gen = ld_acquire_u32(&bar[1]);
  for (int i = 0; i < iters; ++i) grid_barrier<VARIANT>(bar, gen);
}

template <int V>
float run(unsigned* bar, int grid, int iters) {
  cudaMemset(bar, 0, 64);
  void* args[] = {&bar, &iters};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchCooperativeKernel((void*)k<V>, grid, 256, args, 0, 0);
  cudaMemset(bar, 0, 64);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)k<V>, grid, 256, args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / iters;
}

int main() {
  unsigned* bar;
  cudaMalloc(&bar, 64);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int g : {nsm, 2 * nsm}) {
    printf("grid %d: sleep-spin %.2f us, spin %.2f us, release-counter %.2f us\n", g,
           run<0>(bar, g, 2000), run<1>(bar, g, 2000), run<2>(bar, g, 2000));
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
