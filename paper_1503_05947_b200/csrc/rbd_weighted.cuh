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
static __global__ void __launch_bounds__(kThreads) k_colsq_diag(const double* __restrict__ X, long long ldx,
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
static __global__ void __launch_bounds__(kThreads) k_diag_vec(const double* __restrict__ Y, long long m,
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

// Two dot products per column in one pass over a (chunk, 4-column) tile:
//   partial[s][j] = v . x_j,  partial2[s][j] = v2 . x_j  over the rows of chunk s.
// Same thread -> row layout, per-thread fma order (groups ascending, .x then
// .y) and reduction tree as sweep_tiles<VEC, MODE_DOT>, so `partial` is
// bit-identical to the identity sweep's; out-of-range rows load 0.
// ALOAD: LOAD_STREAM (X) or LOAD_CG (Y, written inside the persistent loop);
// VCOH: the vectors are read L2-coherently (written earlier in the same launch).
template <int VEC, int ALOAD = LOAD_STREAM, bool VCOH = false, int UB = 2>
__device__ __forceinline__ void sweep_tile_dot2(const double* __restrict__ A, long long lda,
                                                long long m, long long ncols,
                                                const double* __restrict__ v,
                                                const double* __restrict__ v2,
                                                double* __restrict__ partial,
                                                double* __restrict__ partial2, long long pstride,
                                                long long tile, double (*red)[2 * kCols]) {
  const long long G = (ncols + kCols - 1) / kCols;
  const long long s = tile / G;
  const long long g = tile - s * G;
  const long long row0 = s * kChunk;
  const long long col0 = g * kCols;
  const long long rows = (m - row0 < kChunk) ? m - row0 : kChunk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int U = kChunk / (VEC * kThreads);
  static_assert(U % UB == 0, "batch must divide the chunk");
  double acc[kCols], acc2[kCols];
  const double* Ac[kCols];
#pragma unroll
  for (int c = 0; c < kCols; ++c) {
    acc[c] = acc2[c] = 0.0;
    const long long cc = (col0 + c < ncols) ? col0 + c : col0;   // clamp (result unused)
    Ac[c] = A + cc * lda + row0;
  }
  const double* vr = v + row0;
  const double* wr = v2 + row0;
#pragma unroll 1
  for (int ub = 0; ub < U; ub += UB) {
    if ((long long)ub * VEC * kThreads >= rows) break;
    double xv[UB][kCols][VEC], yv[UB][VEC], zv[UB][VEC];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const long long e = (long long)(tid + (ub + u) * kThreads) * VEC;
      if (e + VEC <= rows) {
        if constexpr (VEC == 2) {
          const double2 y2 = VCOH ? __ldcg(reinterpret_cast<const double2*>(vr + e)) : ld_keep2(vr + e);
          const double2 z2 = VCOH ? __ldcg(reinterpret_cast<const double2*>(wr + e)) : ld_keep2(wr + e);
          yv[u][0] = y2.x;
          yv[u][VEC - 1] = y2.y;
          zv[u][0] = z2.x;
          zv[u][VEC - 1] = z2.y;
#pragma unroll
          for (int c = 0; c < kCols; ++c) {
            const double2 x2 = ALOAD == LOAD_STREAM ? ld_stream2(Ac[c] + e)
                               : __ldcg(reinterpret_cast<const double2*>(Ac[c] + e));
            xv[u][c][0] = x2.x;
            xv[u][c][VEC - 1] = x2.y;
          }
        } else {
          yv[u][0] = VCOH ? __ldcg(vr + e) : ld_keep1(vr + e);
          zv[u][0] = VCOH ? __ldcg(wr + e) : ld_keep1(wr + e);
#pragma unroll
          for (int c = 0; c < kCols; ++c)
            xv[u][c][0] = ALOAD == LOAD_STREAM ? ld_stream1(Ac[c] + e) : __ldcg(Ac[c] + e);
        }
      } else {
#pragma unroll
        for (int q = 0; q < VEC; ++q) {
          const bool in = e + q < rows;
          yv[u][q] = in ? (VCOH ? __ldcg(vr + e + q) : __ldg(vr + e + q)) : 0.0;
          zv[u][q] = in ? (VCOH ? __ldcg(wr + e + q) : __ldg(wr + e + q)) : 0.0;
#pragma unroll
          for (int c = 0; c < kCols; ++c)
            xv[u][c][q] = in ? (ALOAD == LOAD_STREAM ? __ldcs(Ac[c] + e + q) : __ldcg(Ac[c] + e + q))
                             : 0.0;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < UB; ++u)
#pragma unroll
      for (int c = 0; c < kCols; ++c)
#pragma unroll
        for (int q = 0; q < VEC; ++q) {
          acc[c] = fma(xv[u][c][q], yv[u][q], acc[c]);
          acc2[c] = fma(xv[u][c][q], zv[u][q], acc2[c]);
        }
  }
#pragma unroll
  for (int c = 0; c < kCols; ++c)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], off);
      acc2[c] += __shfl_xor_sync(0xffffffffu, acc2[c], off);
    }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < kCols; ++c) {
      red[warp][c] = acc[c];
      red[warp][kCols + c] = acc2[c];
    }
  }
  __syncthreads();
  if (tid < 2 * kCols) {
    const int c = tid % kCols;
    if (col0 + c < ncols) {
      double sum = red[0][tid];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) sum += red[w][tid];
      (tid < kCols ? partial : partial2)[s * pstride + col0 + c] = sum;
    }
  }
  __syncthreads();
}

// sweep_tile_dot2 for the persistent weighted loop's X tiles (VEC 2): the two
// vectors travel by per-thread cp.async into this thread's own shared-memory
// slots (no CTA barrier needed), so registers hold only X while the loads are
// in flight and a batch keeps UB x kCols 16-byte X loads outstanding (UB 4:
// the identity sweep's depth). Same row layout, fma order and reduction as
// sweep_tile_dot2, hence the same bits. sv: [UB][2][kThreads] double2.
constexpr int kSvUB = 4;
constexpr int kSvBytes = kSvUB * 2 * kThreads * 16;   // 32 KiB per CTA
// The persistent loop passes the tile as (chunk s, group g) — no 64-bit
// division per tile — and TRAIL = false: its claim barrier orders `red` for the
// next tile, and it adds a barrier itself where a finalisation may read these
// partials. The two 4-column reductions run as one transposed 8-way butterfly
// (warp_cols_to_red: 9 shuffles per warp instead of 40, the same sums bit for
// bit).
template <int ALOAD = LOAD_STREAM, int UB = kSvUB, bool TRAIL = true>
__device__ __forceinline__ void sweep_tile_dot2_sv(const double* __restrict__ A, long long lda,
                                                   long long m, long long ncols,
                                                   const double* __restrict__ v,
                                                   const double* __restrict__ v2,
                                                   double* __restrict__ partial,
                                                   double* __restrict__ partial2, long long pstride,
                                                   long long s, long long g,
                                                   double (*red)[2 * kCols],
                                                   double2* __restrict__ sv) {
  constexpr int VEC = 2;
  const long long row0 = s * kChunk;
  const long long col0 = g * kCols;
  const long long rows = (m - row0 < kChunk) ? m - row0 : kChunk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int U = kChunk / (VEC * kThreads);
  static_assert(U % UB == 0, "batch must divide the chunk");
  double acc[kCols], acc2[kCols];
  const double* Ac[kCols];
#pragma unroll
  for (int c = 0; c < kCols; ++c) {
    acc[c] = acc2[c] = 0.0;
    const long long cc = (col0 + c < ncols) ? col0 + c : col0;   // clamp (result unused)
    Ac[c] = A + cc * lda + row0;
  }
  const double* vr = v + row0;
  const double* wr = v2 + row0;
#pragma unroll 1
  for (int ub = 0; ub < U; ub += UB) {
    if ((long long)ub * VEC * kThreads >= rows) break;
    double2 xv[UB][kCols];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const long long e = (long long)(tid + (ub + u) * kThreads) * VEC;
      double2* s0 = sv + (2 * u) * kThreads + tid;
      double2* s1 = sv + (2 * u + 1) * kThreads + tid;
      if (e + VEC <= rows) {
        const unsigned a0 = (unsigned)__cvta_generic_to_shared(s0);
        const unsigned a1 = (unsigned)__cvta_generic_to_shared(s1);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a0), "l"(vr + e) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a1), "l"(wr + e) : "memory");
#pragma unroll
        for (int c = 0; c < kCols; ++c)
          xv[u][c] = ALOAD == LOAD_STREAM ? ld_stream2(Ac[c] + e)
                                          : __ldcg(reinterpret_cast<const double2*>(Ac[c] + e));
      } else {
        const bool in0 = e < rows, in1 = e + 1 < rows;
        *s0 = make_double2(in0 ? __ldcg(vr + e) : 0.0, in1 ? __ldcg(vr + e + 1) : 0.0);
        *s1 = make_double2(in0 ? __ldcg(wr + e) : 0.0, in1 ? __ldcg(wr + e + 1) : 0.0);
#pragma unroll
        for (int c = 0; c < kCols; ++c)
          xv[u][c] = ALOAD == LOAD_STREAM
                         ? make_double2(in0 ? __ldcs(Ac[c] + e) : 0.0, in1 ? __ldcs(Ac[c] + e + 1) : 0.0)
                         : make_double2(in0 ? __ldcg(Ac[c] + e) : 0.0, in1 ? __ldcg(Ac[c] + e + 1) : 0.0);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const double2 y2 = sv[(2 * u) * kThreads + tid];
      const double2 z2 = sv[(2 * u + 1) * kThreads + tid];
#pragma unroll
      for (int c = 0; c < kCols; ++c) {
        acc[c] = fma(xv[u][c].x, y2.x, acc[c]);
        acc2[c] = fma(xv[u][c].x, z2.x, acc2[c]);
        acc[c] = fma(xv[u][c].y, y2.y, acc[c]);
        acc2[c] = fma(xv[u][c].y, z2.y, acc2[c]);
      }
    }
  }
  {
    double acc8[2 * kCols];
#pragma unroll
    for (int c = 0; c < kCols; ++c) {
      acc8[c] = acc[c];
      acc8[kCols + c] = acc2[c];
    }
    warp_cols_to_red<2 * kCols>(acc8, red, lane, warp);
  }
  __syncthreads();
  if (tid < 2 * kCols) {
    const int c = tid % kCols;
    if (col0 + c < ncols) {
      double sum = red[0][tid];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) sum += red[w][tid];
      (tid < kCols ? partial : partial2)[s * pstride + col0 + c] = sum;
    }
  }
  if constexpr (TRAIL) __syncthreads();
}

// One X pass for both new rows: T row partials (xi . x_j, decompose.cpp:93) and
// YAX row partials ((A xi) . x_j, workspace.cpp:66).
template <int VEC>
__global__ void __launch_bounds__(kThreads, 2) k_sweep_diag(const double* __restrict__ X,
                                                            long long ldx, long long m, long long n,
                                                            const double* __restrict__ Y,
                                                            const double* __restrict__ axi,
                                                            double* __restrict__ partial,
                                                            double* __restrict__ partial2,
                                                            const DevState* st) {
  if (st->done) return;
  __shared__ double red[kWarps][2 * kCols];
  const double* xi = Y + st->d * m;
  const long long ntiles = ((m + kChunk - 1) / kChunk) * ((n + kCols - 1) / kCols);
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x)
    sweep_tile_dot2<VEC>(X, ldx, m, n, xi, axi, partial, partial2, n, t, red);
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
// CTA = 32 columns; g_j = YAY[d,0:d] . T[0:d,j] is split over the 8 warps
// (l = warp, warp+8, ...; coalesced T rows) and combined in warp order.
constexpr int kFdCols = 32;
static __global__ void __launch_bounds__(kThreads) k_finalize_diag(FinalizeDiagArgs a) {
  const FinalizeArgs& f = a.f;
  if (f.st->done) return;
  __shared__ Rec smr[kWarps];
  __shared__ int is_last;
  __shared__ double yydd_s;
  __shared__ double gpart[kWarps][kFdCols];
  const long long n = f.n;
  const long long k = f.st->d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < a.yy_np; ++b) s += a.yy_part[b];
    yydd_s = s;
  }
  double bv = -1.0;  // workspace.cpp:105
  long long bj = 0x7fffffffffffffffLL;
  const long long nb = (n + kFdCols - 1) / kFdCols;
  for (long long blk = blockIdx.x; blk < nb; blk += gridDim.x) {
    const long long j = blk * kFdCols + lane;
    const bool col = j < n;
    double gp = 0.0;
    if (col) {
      long long l = warp;
      for (; l + 3 * kWarps < k; l += 4 * kWarps) {   // 4 loads in flight per lane
        const double t0 = __ldcg(&f.T[l * n + j]), t1 = __ldcg(&f.T[(l + kWarps) * n + j]);
        const double t2 = __ldcg(&f.T[(l + 2 * kWarps) * n + j]);
        const double t3 = __ldcg(&f.T[(l + 3 * kWarps) * n + j]);
        gp = fma(a.yrow[l], t0, gp);
        gp = fma(a.yrow[l + kWarps], t1, gp);
        gp = fma(a.yrow[l + 2 * kWarps], t2, gp);
        gp = fma(a.yrow[l + 3 * kWarps], t3, gp);
      }
      for (; l < k; l += kWarps) gp = fma(a.yrow[l], __ldcg(&f.T[l * n + j]), gp);
    }
    gpart[warp][lane] = gp;
    __syncthreads();
    if (warp == 0 && col) {
      double g = gpart[0][lane];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) g += gpart[w][lane];
      double t = 0.0, ya = 0.0;
      for (long long s = 0; s < f.S; ++s) {
        t += f.partial[s * n + j];
        ya += a.partial2[s * n + j];
      }
      f.T[k * n + j] = t;
      a.YAX[k * n + j] = ya;
      const double yydd = yydd_s;
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
    __syncthreads();
  }
  finalize_reduce_tail(f, k, bv, bj, smr, &is_last);
}

// ---------------------------------------------------------------------------
// ErrorWorkspace with a diagonal weight (rbd_ws_* on a diagonal workspace;
// workspace.cpp:24-29, 61-79, 84-99, 101-125).
// ---------------------------------------------------------------------------

// out[j] = sum over chunks s of partial[s * n + j] (chunks in order).
static __global__ void k_rowsum(const double* __restrict__ partial, long long S, long long n,
                         double* __restrict__ out) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (long long s = 0; s < S; ++s) t += partial[s * n + j];
    out[j] = t;
  }
}

// YAY row d (workspace.cpp:69-75): yay[d][k] = yay[k][d] = row[k] (k < d),
// yay[d][d] = sum of the xi' A xi partials (in order).
static __global__ void k_yay_row(const double* __restrict__ row, long long d, const double* __restrict__ yy_part,
                          int np, double* __restrict__ yay, long long ld) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < d;
       k += (long long)gridDim.x * blockDim.x) {
    yay[d * ld + k] = row[k];
    yay[k * ld + d] = row[k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < np; ++b) s += yy_part[b];
    yay[d * ld + d] = s;
  }
}

// error_sq (workspace.cpp:84-99) for one column: cross = c . yax[:, j],
// quad = c' yay c (yay == nullptr: identity, quad = ||c||^2).
static __global__ void __launch_bounds__(kThreads) k_error_sq_w(const double* __restrict__ yax, long long n,
                                                         long long d, long long j,
                                                         const double* __restrict__ c,
                                                         const double* __restrict__ yay, long long ld,
                                                         const double* __restrict__ col_sq,
                                                         double* __restrict__ out) {
  __shared__ double sm[kWarps];
  double cross = 0.0, quad = 0.0;
  for (long long k = threadIdx.x; k < d; k += kThreads) {
    cross = fma(c[k], yax[k * n + j], cross);
    double yc = c[k];
    if (yay) {
      yc = 0.0;
      for (long long l = 0; l < d; ++l) yc = fma(yay[k * ld + l], c[l], yc);
    }
    quad = fma(c[k], yc, quad);
  }
  cross = block_sum_fixed<kThreads>(cross, sm);
  quad = block_sum_fixed<kThreads>(quad, sm);
  if (threadIdx.x == 0) {
    const double e2 = col_sq[j] - 2.0 * cross + quad;   // :95-96
    out[0] = e2 > 0.0 ? e2 : 0.0;
  }
}

// residual_scan for a general weight (workspace.cpp:114-122): error_sq of every
// column with c = T[:, j] (T row-major d x n), argmax with smallest-index
// ties, E_cur = sqrt(max(best, 0)) (:123); last-CTA reduction into out.
static __global__ void __launch_bounds__(kThreads) k_scan_T(const double* __restrict__ yax,
                                                     const double* __restrict__ T, long long n,
                                                     long long d, const double* __restrict__ yay,
                                                     long long ld, const double* __restrict__ col_sq,
                                                     Rec* rec, unsigned* counter, Rec* out) {
  __shared__ Rec smr[kWarps];
  __shared__ int is_last;
  double bv = -1.0;
  long long bj = 0x7fffffffffffffffLL;
  for (long long j = blockIdx.x * (long long)kThreads + threadIdx.x; j < n;
       j += (long long)gridDim.x * kThreads) {
    double cross = 0.0, quad = 0.0;
    for (long long k = 0; k < d; ++k) {
      const double ck = T[k * n + j];
      cross = fma(ck, yax[k * n + j], cross);
      double yc = ck;
      if (yay) {
        yc = 0.0;
        for (long long l = 0; l < d; ++l) yc = fma(yay[k * ld + l], T[l * n + j], yc);
      }
      quad = fma(ck, yc, quad);
    }
    double e2 = col_sq[j] - 2.0 * cross + quad;
    e2 = e2 > 0.0 ? e2 : 0.0;
    if (rec_better(e2, j, bv, bj)) {
      bv = e2;
      bj = j;
    }
  }
  block_argmax<kThreads>(bv, bj, smr);
  if (threadIdx.x == 0) {
    rec[blockIdx.x] = Rec{bv, bj};
    __threadfence();
    is_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  bv = -1.0;
  bj = 0x7fffffffffffffffLL;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += kThreads) {
    const Rec rr{__ldcg(&rec[b].v), __ldcg(&rec[b].j)};
    if (rec_better(rr.v, rr.j, bv, bj)) {
      bv = rr.v;
      bj = rr.j;
    }
  }
  block_argmax<kThreads>(bv, bj, smr);
  if (threadIdx.x == 0) {
    *counter = 0u;
    if (bj == 0x7fffffffffffffffLL) bj = 0;
    out[0] = Rec{sqrt(bv > 0.0 ? bv : 0.0), bj};
  }
}

}  // namespace rbdk
