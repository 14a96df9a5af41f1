// rbd_weighted.cuh — the greedy loop with a diagonal weight A = diag(a)
// (reference weight.cpp:11-21,78-121,
// workspace.cpp:24-29,61-79,84-99,114-122).
//
// In the reference the weight changes only the error bookkeeping: Y stays
// Euclidean-orthonormal and T = Y'X (mgs_project and decompose.cpp:93 are
// weight-free), while the greedy scan evaluates, for every column j,
//   e2_j = col_sq_A[j] - 2 c.yax[:,j] + c' (Y'AY) c,   c = T[:,j]
// from scratch (O(n d^2) per step). Here the two sums are carried per column
// and extended by one basis vector per step:
//   cross_j += T[d,j] * YAX[d,j]
//   quad_j  += 2 T[d,j] g_j + YAY[d,d] T[d,j]^2,   g_j = YAY[d,0:d] . T[0:d,j]
// with YAX[d,j] = (A xi).x_j from the same X pass as T[d,j], YAY[d,0:d] =
// Y'(A xi) from one pass over Y and YAY[d,d] = xi'A xi.
#pragma once

#include "rbd_device.cuh"

namespace rbdk {

// col_sq_A[j] = max(sum_i x_ij^2 a_i, 0) (workspace.cpp:24-29,37); one CTA per
// column, fixed per-thread row order and a fixed reduction tree.
__global__ void __launch_bounds__(kThreads) k_colsq_diag(const double* __restrict__ X, long long ldx,
                                                         long long m, long long n,
                                                         const double* __restrict__ diag,
                                                         double* __restrict__ colsq_a) {
  __shared__ double sm[kWarps];
  for (long long j = blockIdx.x; j < n; j += gridDim.x) {
    const double* x = X + j * ldx;
    double acc = 0.0;
    for (long long i = threadIdx.x; i < m; i += kThreads) {
      const double v = x[i];
      acc = fma(v * v, diag[i], acc);
    }
    acc = block_sum_fixed<kThreads>(acc, sm);
    if (threadIdx.x == 0) colsq_a[j] = acc > 0.0 ? acc : 0.0;
  }
}

// a_xi = a o xi (weight.cpp:83) for the vector just written to Y[:, st->d];
// yy_part[b] = this CTA's share of xi' A xi (workspace.cpp:75). Fixed grid.
__global__ void __launch_bounds__(kThreads) k_diag_vec(const double* __restrict__ Y, long long m,
                                                       const double* __restrict__ diag,
                                                       double* __restrict__ axi,
                                                       double* __restrict__ yy_part,
                                                       const DevState* st) {
  if (st->done) return;
  __shared__ double sm[kWarps];
  const double* xi = Y + st->d * m;
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < m;
       i += (long long)gridDim.x * kThreads) {
    const double x = xi[i];
    const double v = diag[i] * x;
    axi[i] = v;
    acc = fma(v, x, acc);
  }
  acc = block_sum_fixed<kThreads>(acc, sm);
  if (threadIdx.x == 0) yy_part[blockIdx.x] = acc;
}

// One X pass for both new rows: partial[s][j] = xi . x_j over chunk s (T row,
// decompose.cpp:93) and partial2[s][j] = (A xi) . x_j (YAX row, workspace.cpp:66).
// The tile is swept twice back to back; the second sweep reads it from L2.
template <int VEC>
__global__ void __launch_bounds__(kThreads, 2) k_sweep_diag(const double* __restrict__ X,
                                                            long long ldx, long long m, long long n,
                                                            const double* __restrict__ Y,
                                                            const double* __restrict__ axi,
                                                            double* __restrict__ partial,
                                                            double* __restrict__ partial2,
                                                            const DevState* st) {
  if (st->done) return;
  __shared__ double red[kWarps][kCols];
  unsigned nf = 0, nz = 0;
  const double* xi = Y + st->d * m;
  const long long ntiles = ((m + kChunk - 1) / kChunk) * ((n + kCols - 1) / kCols);
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    sweep_tiles<VEC, MODE_DOT, LOAD_NC>(X, ldx, m, n, xi, partial, n, t, 1LL << 40, red, nf, nz);
    sweep_tiles<VEC, MODE_DOT, LOAD_NC>(X, ldx, m, n, axi, partial2, n, t, 1LL << 40, red, nf, nz);
  }
}

struct FinalizeDiagArgs {
  FinalizeArgs f;            // partial (T row), T, st, rec, counter, history, cbuf, col_sq (Euclidean)
  const double* partial2;    // YAX row partials
  double* YAX;               // row-major d_max x n
  const double* yrow;        // YAY[d, 0:d]
  const double* yy_part;     // xi' A xi partials
  int yy_np;
  double* cross;             // per column: sum_k T[k,j] YAX[k,j]
  double* quad;              // per column: T[:,j]' YAY T[:,j]
  const double* colsq_a;     // ||x_j||_A^2
};

// K3 with a diagonal weight: new T and YAX rows, the carried cross/quad sums,
// e2_j = max(col_sq_A - 2 cross + quad, 0) (workspace.cpp:88-97), the argmax
// with smallest-index ties (workspace.cpp:114-122) and the stop test.
__global__ void __launch_bounds__(kThreads) k_finalize_diag(FinalizeDiagArgs a) {
  const FinalizeArgs& f = a.f;
  if (f.st->done) return;
  __shared__ Rec smr[kWarps];
  __shared__ int is_last;
  __shared__ double yydd_s;
  const long long n = f.n;
  const long long k = f.st->d;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < a.yy_np; ++b) s += a.yy_part[b];
    yydd_s = s;
  }
  __syncthreads();
  const double yydd = yydd_s;
  double bv = -1.0;  // workspace.cpp:105
  long long bj = 0x7fffffffffffffffLL;
  for (long long j = blockIdx.x * (long long)kThreads + threadIdx.x; j < n;
       j += (long long)gridDim.x * kThreads) {
    double t = 0.0, ya = 0.0;
    for (long long s = 0; s < f.S; ++s) {
      t += f.partial[s * n + j];
      ya += a.partial2[s * n + j];
    }
    f.T[k * n + j] = t;
    a.YAX[k * n + j] = ya;
    double g = 0.0;
    for (long long l = 0; l < k; ++l) g = fma(a.yrow[l], f.T[l * n + j], g);
    const double cr = a.cross[j] + t * ya;
    const double qd = a.quad[j] + (2.0 * t * g + yydd * t * t);
    a.cross[j] = cr;
    a.quad[j] = qd;
    double e2 = a.colsq_a[j] - 2.0 * cr + qd;
    e2 = e2 > 0.0 ? e2 : 0.0;
    if (rec_better(e2, j, bv, bj)) {
      bv = e2;
      bj = j;
    }
  }
  finalize_reduce_tail(f, k, bv, bj, smr, &is_last);
}

}  // namespace rbdk
