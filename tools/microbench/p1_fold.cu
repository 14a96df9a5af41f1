// Microbenchmark: can P1 form its CTA's share of p_k = Y'w1_k from the row
// block it just read (second read served by L2), instead of the separate
// full-height Y'w1 groups that read Y from HBM a second time when Y does not
// fit L2 (C2: Y up to 4 GiB)? Per row block (NH halves of 64 rows; a lane owns
// a 16-byte row pair, the 8/NH warps of a half split the columns):
//   pass 1  acc = Y[block, 0:k] c  -> w1 = x - acc (the loop's P1 arithmetic)
//   pass 2  p_share[l] += sum_rows Y[row, l] w1[row]  (re-read of the block;
//           a 16-column transposing butterfly per warp: one shuffle per column)
// Compared with P1 alone (pass 1) and with pass 2 streamed from HBM (the cost
// the fold removes). HINT: pass-1 loads with L2::evict_last, pass-2 loads
// with L2::evict_first.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 p1_fold.cu -o p1_fold
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kT = 256;
constexpr int kL = 16;   // loads in flight per lane per batch

__device__ __forceinline__ double2 ld2(const double* p, int hint) {
  double2 v;
  if (hint == 1) {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  } else if (hint == 2) {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  } else {
    v = __ldcg(reinterpret_cast<const double2*>(p));
  }
  return v;
}

// one level of the transposing butterfly: S values per lane -> S/2... (keeps
// the half selected by lane bit BIT, adds the partner's copy of it)
template <int S, int BIT>
__device__ __forceinline__ void bfly(double* t, int lane) {
  const bool upper = (lane & BIT) != 0;
#pragma unroll
  for (int q = 0; q < S; ++q) {
    const double send = upper ? t[q] : t[q + S];
    const double keep = upper ? t[q + S] : t[q];
    t[q] = keep + __shfl_xor_sync(0xffffffffu, send, BIT);
  }
}

// MODE 0: pass 1 only; 1: pass 1 + pass 2 (fold); 2: pass 2 only (w1 = given)
template <int NH, int MODE, int HINT>
__global__ void __launch_bounds__(kT, 2) k_fold(const double* __restrict__ Y, long long m, int k,
                                               const double* __restrict__ c,
                                               const double* __restrict__ x, double* w,
                                               double* pshare) {
  constexpr int kPW = 8 / NH;          // warps per half
  constexpr int R = 64 * NH;           // rows per block
  __shared__ double red[8][64];
  __shared__ double w1s[R];
  __shared__ double psh[NH][1024];
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long lo = ((m * cta / G) + 1) & ~1LL, hi = (cta + 1 == G) ? m : (((m * (cta + 1) / G) + 1) & ~1LL);
  const int half = warp / kPW, wh = warp % kPW;
  for (int l = tid; l < NH * 1024; l += kT) (&psh[0][0])[l] = 0.0;
  __syncthreads();
  for (long long rb = lo; rb < hi; rb += R) {
    const long long i0 = rb + half * 64 + 2 * lane;
    const bool ok2 = i0 + 1 < hi;
    if (MODE != 2) {
      double a0 = 0.0, a1 = 0.0;
      if (ok2) {
        const double* yp = Y + i0 + (long long)wh * m;
        for (int l = wh; l < k; l += kL * kPW) {
          double2 v[kL];
#pragma unroll
          for (int q = 0; q < kL; ++q)
            v[q] = (l + q * kPW < k) ? ld2(yp + (long long)q * kPW * m, HINT ? 1 : 0) : make_double2(0, 0);
#pragma unroll
          for (int q = 0; q < kL; ++q) {
            const double cc = c[(l + q * kPW) & 1023];
            a0 = fma(v[q].x, cc, a0);
            a1 = fma(v[q].y, cc, a1);
          }
          yp += (long long)kL * kPW * m;
        }
      }
      red[warp][2 * lane] = a0;
      red[warp][2 * lane + 1] = a1;
      __syncthreads();
      if (wh == 0 && ok2) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          double s = red[half * kPW][2 * lane + v];
#pragma unroll
          for (int ww = 1; ww < kPW; ++ww) s += red[half * kPW + ww][2 * lane + v];
          const double w1 = x[i0 + v] - s;
          w[i0 + v] = w1;
          w1s[half * 64 + 2 * lane + v] = w1;
        }
      }
      __syncthreads();
    } else {
      if (wh == 0) {
        w1s[half * 64 + 2 * lane] = ok2 ? x[i0] : 0.0;
        w1s[half * 64 + 2 * lane + 1] = ok2 ? x[i0 + 1] : 0.0;
      }
      __syncthreads();
    }
    if (MODE != 0) {
      constexpr int kStep = kL * kPW;
      const int nb = (k - wh + kStep - 1) / kStep;   // batches of this warp
      const double wa = ok2 ? w1s[half * 64 + 2 * lane] : 0.0;
      const double wb = ok2 ? w1s[half * 64 + 2 * lane + 1] : 0.0;
      const double* yb = Y + (ok2 ? i0 : lo);
      for (int bi = 0; bi < nb; ++bi) {
        const int l = wh + (MODE == 3 ? nb - 1 - bi : bi) * kStep;   // MODE 3: most recently read first
        const double* yp = yb + (long long)l * m;
        double t[kL];
#pragma unroll
        for (int q = 0; q < kL; ++q) {
          const double2 v = (l + q * kPW < k) ? ld2(yp + (long long)q * kPW * m, HINT ? 2 : 0) : make_double2(0, 0);
          t[q] = fma(v.y, wb, v.x * wa);
        }
        // transposing butterfly: 16 values per lane -> lane L holds column
        // q(L) = (L>>1)&15 summed over all 32 lanes (L and L^1 agree)
        bfly<8, 16>(t, lane);
        bfly<4, 8>(t, lane);
        bfly<2, 4>(t, lane);
        bfly<1, 2>(t, lane);
        t[0] += __shfl_xor_sync(0xffffffffu, t[0], 1);
        const int q = (((lane >> 4) & 1) << 3) | (((lane >> 3) & 1) << 2) | (((lane >> 2) & 1) << 1) | ((lane >> 1) & 1);
        const int col = l + q * kPW;
        if ((lane & 1) == 0 && col < k) psh[half][col] += t[0];
      }
    }
    __syncthreads();
  }
  for (int l = tid; l < k; l += kT) {
    double s = 0.0;
#pragma unroll
    for (int h = 0; h < NH; ++h) s += psh[h][l];
    pshare[(long long)cta * 1024 + l] = s;
  }
}

int main(int argc, char** argv) {
  const long long m = argc > 1 ? atoll(argv[1]) : (1 << 20);
  double *Y, *c, *x, *w, *ps;
  const int kmax = 1024;
  cudaMalloc(&Y, sizeof(double) * m * kmax / 2);
  cudaMalloc(&c, sizeof(double) * 1024);
  cudaMalloc(&x, sizeof(double) * m);
  cudaMalloc(&w, sizeof(double) * m);
  cudaMalloc(&ps, sizeof(double) * 1024 * 1024);
  cudaMemset(Y, 0x3f, sizeof(double) * m * kmax / 2);
  cudaMemset(c, 0, sizeof(double) * 1024);
  cudaMemset(x, 0, sizeof(double) * m);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* flush;
  const size_t fb = 512ull << 20;
  cudaMalloc(&flush, fb);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int k : {128, 256, 384, 512}) {
    const double bytes = (double)m * k * 8;
    auto timeit = [&](auto launch, const char* name) {
      launch();
      cudaDeviceSynchronize();
      float best = 1e30f;
      for (int r = 0; r < 7; ++r) {
        cudaMemsetAsync(flush, r, fb);   // L2 cold for Y
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      cudaError_t e = cudaGetLastError();
      printf("k=%4d %-40s %8.3f ms  %7.1f GB/s (one Y read)  %s\n", k, name, best, bytes / best / 1e6,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
#define T(NH, MODE, HINT, NAME) timeit([&] { k_fold<NH, MODE, HINT><<<2 * nsm, kT>>>(Y, m, k, c, x, w, ps); }, NAME)
    T(2, 0, 0, "P1 only, 128-row blocks");
    T(2, 2, 0, "Y'w pass from HBM, 128-row blocks");
    T(2, 1, 0, "P1 + fold, 128-row blocks");
    T(2, 1, 1, "P1 + fold, 128-row, L2 hints");
    T(1, 0, 0, "P1 only, 64-row blocks");
    T(1, 1, 0, "P1 + fold, 64-row blocks");
    T(1, 1, 1, "P1 + fold, 64-row, L2 hints");
    T(1, 3, 0, "P1 + fold, 64-row, reversed");
    T(2, 3, 0, "P1 + fold, 128-row, reversed");
  }
  return 0;
}
