// rbd_classify.cuh — batched Classifier::predict (
// reference proj/src/classify.cpp:22-34, classify.hpp:14-21).
//
// For query coordinates c_q = Y'v_q (K5, DMMA) the reference scans the training
// coordinates T (d x n_train, = model.T) for the smallest squared Euclidean
// distance ||T[:,j] - c_q||^2, computed in difference form, strict '<', so the
// earliest column wins ties. Here one CTA evaluates a 64-query x 64-column tile
// of those distances (difference form, fp64 FMA, k ascending) with operands
// staged in shared memory, keeps a running (distance, column) minimum per query
// across the column tiles of its split, and the splits are combined by a
// second tiny kernel. The expansion ||t||^2 - 2 t.c + ||c||^2 (a GEMM) is not
// used: it cancels for near neighbours and would reorder near-ties.
#pragma once

#include "rbd_device.cuh"

namespace rbdk {

constexpr int kNnTile = 64;   // training columns per tile and queries per CTA
constexpr int kNnK = 16;      // coordinates staged per step
constexpr int kNnPad = 1;     // smem padding (doubles) against bank conflicts

struct NnRec {
  double v;
  long long j;
};

__device__ __forceinline__ bool nn_better(double av, long long aj, double bv, long long bj) {
  return av < bv || (av == bv && aj < bj);   // classify.cpp:27-31 (strict <, ascending j)
}

// C: d x Q coordinates, column-major (ld ldc). Tt: d x n_tr, row-major (T[k*n_tr + j]).
// out[split * Q + q] = best (distance, column) of query q over the columns of
// split `blockIdx.y` (cols_per_split, a multiple of kNnTile).
static __global__ void __launch_bounds__(kThreads) k_nearest(const double* __restrict__ C, long long ldc,
                                                      const double* __restrict__ Tt,
                                                      long long n_tr, long long d, long long Q,
                                                      long long cols_per_split,
                                                      NnRec* __restrict__ out) {
  __shared__ double Ts[kNnK][kNnTile + kNnPad];
  __shared__ double Cs[kNnK][kNnTile + kNnPad];
  const int tid = threadIdx.x;
  const int tx = tid & 15;        // training sub-columns tx, tx+16, tx+32, tx+48
  const int ty = tid >> 4;        // queries ty, ty+16, ty+32, ty+48
  const long long q0 = (long long)blockIdx.x * kNnTile;
  const long long jb = (long long)blockIdx.y * cols_per_split;
  const long long je = (jb + cols_per_split < n_tr) ? jb + cols_per_split : n_tr;
  double bv[4];
  long long bj[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    bv[l] = __longlong_as_double(0x7ff0000000000000LL);   // +inf
    bj[l] = 0x7fffffffffffffffLL;
  }
  for (long long j0 = jb; j0 < je; j0 += kNnTile) {
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int l = 0; l < 4; ++l) acc[i][l] = 0.0;
    for (long long k0 = 0; k0 < d; k0 += kNnK) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int idx = tid + kThreads * r;
        // training tile: rows k0..k0+15 of T, 64 contiguous columns each
        const int kk = idx / kNnTile, jj = idx % kNnTile;
        const long long k = k0 + kk, j = j0 + jj;
        Ts[kk][jj] = (k < d && j < je) ? __ldg(&Tt[k * n_tr + j]) : 0.0;
        // query tile: 16 contiguous coordinates of each of 64 query columns
        const int kq = idx % kNnK, qq = idx / kNnK;
        const long long kc = k0 + kq, q = q0 + qq;
        Cs[kq][qq] = (kc < d && q < Q) ? __ldg(&C[q * ldc + kc]) : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kNnK; ++kk) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = Ts[kk][tx + 16 * i];
#pragma unroll
        for (int l = 0; l < 4; ++l) b[l] = Cs[kk][ty + 16 * l];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            const double df = a[i] - b[l];
            acc[i][l] = fma(df, df, acc[i][l]);
          }
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {   // ascending column within the thread
      const long long j = j0 + tx + 16 * i;
      if (j < je) {
#pragma unroll
        for (int l = 0; l < 4; ++l)
          if (nn_better(acc[i][l], j, bv[l], bj[l])) {
            bv[l] = acc[i][l];
            bj[l] = j;
          }
      }
    }
  }
  // combine the 16 column lanes of each query (lanes tx = 0..15 of a half-warp)
#pragma unroll
  for (int l = 0; l < 4; ++l) {
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv[l], off);
      const long long oj = __shfl_xor_sync(0xffffffffu, bj[l], off);
      if (nn_better(ov, oj, bv[l], bj[l])) {
        bv[l] = ov;
        bj[l] = oj;
      }
    }
    const long long q = q0 + ty + 16 * l;
    if (tx == 0 && q < Q) out[(long long)blockIdx.y * Q + q] = NnRec{bv[l], bj[l]};
  }
}

// best[q] / dist[q] = the minimum over the splits (order-independent total order).
static __global__ void k_nearest_reduce(const NnRec* __restrict__ part, long long Q, int nsplit,
                                 long long* __restrict__ best, double* __restrict__ dist) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < Q;
       q += (long long)gridDim.x * blockDim.x) {
    NnRec b = part[q];
    for (int s = 1; s < nsplit; ++s) {
      const NnRec r = part[(long long)s * Q + q];
      if (nn_better(r.v, r.j, b.v, b.j)) b = r;
    }
    best[q] = b.j;
    if (dist) dist[q] = b.v;
  }
}

}  // namespace rbdk
