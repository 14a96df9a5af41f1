// rbd_device.cuh — device-side data structures and kernels of the B200 RBD
// greedy loop. Written for sm_100a (B200); see DESIGN.md for the data layout
// and the roofline of each kernel.
//
// Kernel map (reference function each one replaces):
//   k_sweep<MODE_INIT>   K1  workspace_init col_sq + allFinite + zero test
//                            (workspace.cpp:21-23, decompose.cpp:57,63,70)
//   k_sweep<MODE_DOT>    K2  T.row(d) = xi'X and workspace_extend's X'xi
//                            (decompose.cpp:93, workspace.cpp:51) — one X pass,
//                            chunk partials; also Y'w for the reorth pass
//   k_finalize           K3  residual_sq -= row^2, clamp, residual_scan argmax,
//                            stop test (workspace.cpp:52-53,107-113,123;
//                            decompose.cpp:87,98-101)
//   k_ext_gemv_n / k_ext_* K4 mgs_project (decompose.cpp:12-33) as CGS with the
//                            stored coefficients T[:,j*] plus the reference's
//                            conditional second pass
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rbdk {

// ---- tiling constants (the per-column summation order depends on these and
//      on m only, never on n, the grid or the number of GPUs) ----
constexpr int kThreads = 256;      // sweep CTA size
constexpr int kChunk = 4096;       // rows per sweep tile (32 KiB per column in fp64)
constexpr int kCols = 4;           // columns per sweep tile
constexpr int kWarps = kThreads / 32;
constexpr int kGemvRows = 64;      // rows per GEMV-N CTA
constexpr int kGemvSplit = 4;      // l-splits per row in GEMV-N (kThreads = 64*4)
constexpr int kCoefTile = 2048;    // coefficients staged in smem per pass

enum Gate : int { GATE_NONE = 0, GATE_LIVE = 1, GATE_REORTH = 2 };
enum SweepMode : int { MODE_INIT = 0, MODE_DOT = 1 };
// load flavour of the swept matrix: read-only path, streaming, or L2-coherent
enum LoadKind : int { LOAD_NC = 0, LOAD_STREAM = 1, LOAD_CG = 2 };

// Device-resident loop state. Every per-step kernel reads it, so one captured
// CUDA graph of G steps is valid for any step index.
struct DevState {
  long long d;            // accepted basis vectors so far (the reference's d)
  long long jstar;        // global index of the column to extend with next
  long long jlocal;       // local index of that column on this rank (-1: not owned)
  long long d_max;
  double e_cur;           // last E_cur
  double eps_R;
  double breakdown_tol;
  double xnorm2;          // ||x_{j*}||^2 (entry norm^2, decompose.cpp:18)
  double w1n2;            // ||w||^2 after the first pass
  double wnorm;           // final norm (MgsResult::residual_norm)
  int done;               // loop finished
  int breakdown;          // finished by an orthogonalisation breakdown
  int reorth;             // second pass active this step
  int cfg_reorth;         // RbdConfig::reorthogonalize
  unsigned flags_nonfinite;
  unsigned flags_nonzero;
  unsigned long long max_colsq_bits;  // max_j col_sq (as ordered bits, >= 0)
  int rank_owner;         // multi-GPU: rank owning jstar
  int pending;            // column d-1 of Y not yet materialised (fused path)
  unsigned counter_b;     // last-CTA counter of k_ext_reduce
  unsigned pad2;
};

struct Rec {            // max-loc record: value desc, index asc (workspace.cpp:109)
  double v;
  long long j;
};

__device__ __forceinline__ bool rec_better(double av, long long aj, double bv, long long bj) {
  return av > bv || (av == bv && aj < bj);
}

__device__ __forceinline__ bool gate_skip(const DevState* st, int gate) {
  if (gate == GATE_NONE) return false;
  if (st->done) return true;
  if (gate == GATE_REORTH && !st->reorth) return true;
  return false;
}

// Streaming load (X is read once per step and must not evict Y/T/r from L2).
// Load-batch fence. ptxas may consume the first loads of a batch before it
// has issued the rest when registers are tight, and the warp then waits a
// full memory latency before issuing the remaining loads. Routing the
// batch's vector values through a select on an XOR of every loaded value
// makes each FMA of the batch depend on all of the batch's loads, so they are
// all issued first. The select never fires (c_batch_fence_never is 0, which
// ptxas cannot know), so the values and their bits are unchanged. Used where
// SASS showed split batches (the sharded loop: C2 at world 1 3310 -> 3254 ms).
__constant__ int c_batch_fence_never = 0;
__device__ __forceinline__ double2 batch_fence(double2 v, unsigned key) {
  const bool never = c_batch_fence_never != 0 && key == 0x5a5a5a5au;
  return never ? make_double2(0.0, 0.0) : v;
}

__device__ __forceinline__ double2 ld_stream2(const double* p) {
  return __ldcs(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double ld_stream1(const double* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_keep2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double ld_keep1(const double* p) { return __ldg(p); }

__device__ __forceinline__ bool is_nonfinite(double x) {
  return (__double_as_longlong(x) & 0x7ff0000000000000LL) == 0x7ff0000000000000LL;
}

// ---------------------------------------------------------------------------
// K1/K2: chunked column dot products.  partial[s*pstride + j] =
//   sum over rows of chunk s of A(i,j)*v(i)   (MODE_DOT)
//   sum over rows of chunk s of A(i,j)^2      (MODE_INIT, plus flags)
// A is m x ncols column-major (lda). Tiles = (chunk s, column group g); the
// grid is persistent (grid-stride over tiles).
// ---------------------------------------------------------------------------
struct SweepArgs {
  const double* A;
  long long lda;
  long long m;
  long long ncols;        // static column count (csel == 0)
  const double* v;        // vector (vsel == 0)
  const double* vbase;    // vsel == 1: v = vbase + st->d * vstride
  long long vstride;
  double* partial;
  long long pstride;
  DevState* st;
  int gate;
  int vsel;
  int csel;               // 1: ncols = st->d (reorth pass over Y)
};

// Tile loop shared by the standalone sweep kernel and the persistent loop.
// KC = columns per tile. A column's chunk sum depends only on the row layout
// (thread -> rows, fma order, reduction tree), never on KC or on how loads are
// batched, so tiles of different widths give bit-identical partials.
// One tile (chunk s, column group g); ends with the partials written by
// tid < KC and no barrier (sweep_tiles adds it; the persistent loop's X tiles
// pass s, g directly instead of a tile index divided again here).
template <int VEC, int MODE, int ALOAD, bool VCOH = false, int KC = kCols, bool FENCE = false>
__device__ __forceinline__ void sweep_tile(const double* __restrict__ A, long long lda,
                                           long long m, long long ncols,
                                           const double* __restrict__ v,
                                           double* __restrict__ partial, long long pstride,
                                           long long s, long long g,
                                           double (*red)[kCols], unsigned& nonfinite,
                                           unsigned& nonzero) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int U = kChunk / (VEC * kThreads);  // element groups per thread per column
  // batch of element groups loaded together: 16 (VEC 2) / 32 (VEC 1) column
  // loads in flight per thread, capped at the whole chunk
  constexpr int UB0 = ((VEC == 2) ? 4 : 8) * (kCols / KC);
  constexpr int UB = UB0 < U ? UB0 : U;
  {
    const long long row0 = s * kChunk;
    const long long col0 = g * KC;
    const long long rows = (m - row0 < kChunk) ? m - row0 : kChunk;
    double acc[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) acc[c] = 0.0;
    const double* vr = (MODE == MODE_DOT) ? v + row0 : nullptr;
    if (VEC == 2 && MODE == MODE_DOT && rows == kChunk && col0 + KC <= ncols &&
        lda <= (1LL << 27)) {
      // full tile (the common case): per batch one base pointer per column,
      // the batch's element groups at immediate offsets (u * 4 KiB), so a load
      // costs no address arithmetic (it was ~35% of the loop's issued
      // instructions: ncu source counters, C2); same loads and fma order as below
      const double* A0 = A + col0 * lda + row0 + 2 * tid;
      const double* V0 = vr + 2 * tid;
#pragma unroll 1
      for (int ub = 0; ub < U; ub += UB) {
        double2 yv[UB];
        double2 xv[UB][KC];
        const double* Ab = A0 + ub * (2 * kThreads);
        const double* Vb = V0 + ub * (2 * kThreads);
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const double* pv = Vb + u * (2 * kThreads);
          yv[u] = VCOH ? __ldcg(reinterpret_cast<const double2*>(pv)) : ld_keep2(pv);
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            const double* pc = Ab + c * lda + u * (2 * kThreads);
            xv[u][c] = ALOAD == LOAD_STREAM ? ld_stream2(pc)
                       : ALOAD == LOAD_CG   ? __ldcg(reinterpret_cast<const double2*>(pc))
                                            : ld_keep2(pc);
          }
        }
        if constexpr (FENCE) {   // every load of the batch before any FMA (batch_fence)
          unsigned key = 0u;
#pragma unroll
          for (int u = 0; u < UB; ++u)
#pragma unroll
            for (int c = 0; c < KC; ++c) key ^= __double2loint(xv[u][c].y);
#pragma unroll
          for (int u = 0; u < UB; ++u) yv[u] = batch_fence(yv[u], key);
        }
#pragma unroll
        for (int u = 0; u < UB; ++u)
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            acc[c] = fma(xv[u][c].x, yv[u].x, acc[c]);
            acc[c] = fma(xv[u][c].y, yv[u].y, acc[c]);
          }
      }
    } else {
    const double* Ac[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      const long long cc = (col0 + c < ncols) ? col0 + c : col0;  // clamp (result unused)
      Ac[c] = A + cc * lda + row0;
    }
    // Batches of UB element groups; a batch lying entirely inside the matrix
    // takes the vector path, the (at most one) straddling batch the
    // predicated path. Both use the same per-thread fma order, out-of-range
    // rows contribute +0, so the result is independent of the path taken.
    constexpr int kBatchRows = UB * VEC * kThreads;
#pragma unroll 1
    for (int ub = 0; ub < U; ub += UB) {
      if ((long long)(ub / UB + 1) * kBatchRows <= rows) {
        if constexpr (VEC == 2) {
          double2 yv[UB];
          double2 xv[UB][KC];
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            const int e = (tid + (ub + u) * kThreads) * 2;
            if constexpr (MODE == MODE_DOT)
              yv[u] = VCOH ? __ldcg(reinterpret_cast<const double2*>(vr + e)) : ld_keep2(vr + e);
#pragma unroll
            for (int c = 0; c < KC; ++c)
              xv[u][c] = ALOAD == LOAD_STREAM ? ld_stream2(Ac[c] + e)
                         : ALOAD == LOAD_CG   ? __ldcg(reinterpret_cast<const double2*>(Ac[c] + e))
                                              : ld_keep2(Ac[c] + e);
          }
#pragma unroll
          for (int u = 0; u < UB; ++u)
#pragma unroll
            for (int c = 0; c < KC; ++c) {
              if constexpr (MODE == MODE_DOT) {
                acc[c] = fma(xv[u][c].x, yv[u].x, acc[c]);
                acc[c] = fma(xv[u][c].y, yv[u].y, acc[c]);
              } else {
                acc[c] = fma(xv[u][c].x, xv[u][c].x, acc[c]);
                acc[c] = fma(xv[u][c].y, xv[u][c].y, acc[c]);
                nonfinite |= is_nonfinite(xv[u][c].x) | is_nonfinite(xv[u][c].y);
                nonzero |= (xv[u][c].x != 0.0) | (xv[u][c].y != 0.0);
              }
            }
        } else {
          double yv[UB];
          double xv[UB][KC];
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            const int e = tid + (ub + u) * kThreads;
            if constexpr (MODE == MODE_DOT) yv[u] = VCOH ? __ldcg(vr + e) : ld_keep1(vr + e);
#pragma unroll
            for (int c = 0; c < KC; ++c)
              xv[u][c] = ALOAD == LOAD_STREAM ? ld_stream1(Ac[c] + e)
                         : ALOAD == LOAD_CG   ? __ldcg(Ac[c] + e)
                                              : ld_keep1(Ac[c] + e);
          }
#pragma unroll
          for (int u = 0; u < UB; ++u)
#pragma unroll
            for (int c = 0; c < KC; ++c) {
              if constexpr (MODE == MODE_DOT) {
                acc[c] = fma(xv[u][c], yv[u], acc[c]);
              } else {
                acc[c] = fma(xv[u][c], xv[u][c], acc[c]);
                nonfinite |= is_nonfinite(xv[u][c]);
                nonzero |= (xv[u][c] != 0.0);
              }
            }
        }
      } else if ((long long)(ub / UB) * kBatchRows < rows) {
        // straddling batch: groups wholly inside take vector loads, the
        // rest predicated loads; identical order either way
#pragma unroll 1
        for (int u = ub; u < ub + UB; ++u) {
          if ((long long)(u + 1) * VEC * kThreads <= rows) {
            const int e = (tid + u * kThreads) * VEC;
            if constexpr (VEC == 2) {
              double2 y2 = make_double2(0.0, 0.0);
              if constexpr (MODE == MODE_DOT)
                y2 = VCOH ? __ldcg(reinterpret_cast<const double2*>(vr + e)) : ld_keep2(vr + e);
              double2 x2[KC];
#pragma unroll
              for (int c = 0; c < KC; ++c)
                x2[c] = ALOAD == LOAD_STREAM ? ld_stream2(Ac[c] + e)
                        : ALOAD == LOAD_CG   ? __ldcg(reinterpret_cast<const double2*>(Ac[c] + e))
                                             : ld_keep2(Ac[c] + e);
#pragma unroll
              for (int c = 0; c < KC; ++c) {
                if constexpr (MODE == MODE_DOT) {
                  acc[c] = fma(x2[c].x, y2.x, acc[c]);
                  acc[c] = fma(x2[c].y, y2.y, acc[c]);
                } else {
                  acc[c] = fma(x2[c].x, x2[c].x, acc[c]);
                  acc[c] = fma(x2[c].y, x2[c].y, acc[c]);
                  nonfinite |= is_nonfinite(x2[c].x) | is_nonfinite(x2[c].y);
                  nonzero |= (x2[c].x != 0.0) | (x2[c].y != 0.0);
                }
              }
            } else {
              double y1 = 0.0;
              if constexpr (MODE == MODE_DOT) y1 = VCOH ? __ldcg(vr + e) : ld_keep1(vr + e);
              double x1[KC];
#pragma unroll
              for (int c = 0; c < KC; ++c)
                x1[c] = ALOAD == LOAD_STREAM ? ld_stream1(Ac[c] + e)
                        : ALOAD == LOAD_CG   ? __ldcg(Ac[c] + e)
                                             : ld_keep1(Ac[c] + e);
#pragma unroll
              for (int c = 0; c < KC; ++c) {
                if constexpr (MODE == MODE_DOT) {
                  acc[c] = fma(x1[c], y1, acc[c]);
                } else {
                  acc[c] = fma(x1[c], x1[c], acc[c]);
                  nonfinite |= is_nonfinite(x1[c]);
                  nonzero |= (x1[c] != 0.0);
                }
              }
            }
            continue;
          }
          if constexpr (VEC == 2) {
            const long long e = (long long)(tid + u * kThreads) * 2;
            double y0 = 0.0, y1 = 0.0;
            if constexpr (MODE == MODE_DOT) {
              if (e < rows) y0 = __ldcg(vr + e);
              if (e + 1 < rows) y1 = __ldcg(vr + e + 1);
            }
#pragma unroll
            for (int c = 0; c < KC; ++c) {
              const double x0 = (e < rows) ? __ldcg(Ac[c] + e) : 0.0;
              const double x1 = (e + 1 < rows) ? __ldcg(Ac[c] + e + 1) : 0.0;
              if constexpr (MODE == MODE_DOT) {
                acc[c] = fma(x0, y0, acc[c]);
                acc[c] = fma(x1, y1, acc[c]);
              } else {
                acc[c] = fma(x0, x0, acc[c]);
                acc[c] = fma(x1, x1, acc[c]);
                nonfinite |= is_nonfinite(x0) | is_nonfinite(x1);
                nonzero |= (x0 != 0.0) | (x1 != 0.0);
              }
            }
          } else {
            const long long e = tid + (long long)u * kThreads;
            double y0 = 0.0;
            if constexpr (MODE == MODE_DOT) {
              if (e < rows) y0 = __ldcg(vr + e);
            }
#pragma unroll
            for (int c = 0; c < KC; ++c) {
              const double x0 = (e < rows) ? __ldcg(Ac[c] + e) : 0.0;
              if constexpr (MODE == MODE_DOT) {
                acc[c] = fma(x0, y0, acc[c]);
              } else {
                acc[c] = fma(x0, x0, acc[c]);
                nonfinite |= is_nonfinite(x0);
                nonzero |= (x0 != 0.0);
              }
            }
          }
        }
      }
    }
    }   // general path
    // CTA reduction in a fixed order: xor-butterfly in the warp, then warps 0..7.
    if constexpr (KC == 4) {
      // the same butterfly tree, transposed: at xor 16 a lane keeps two of
      // the four columns and receives the partner's copies of them, at xor 8
      // one, then xor 4, 2, 1 on that column; every sum has the butterfly's
      // operands in the butterfly's order (x + partner), so the values are the
      // butterfly's bit for bit, with 6 shuffles per warp instead of 20
      const bool h16 = (lane & 16) != 0, h8 = (lane & 8) != 0;
      double k0 = h16 ? acc[2] : acc[0], k1 = h16 ? acc[3] : acc[1];
      const double g0 = h16 ? acc[0] : acc[2], g1 = h16 ? acc[1] : acc[3];
      k0 += __shfl_xor_sync(0xffffffffu, g0, 16);
      k1 += __shfl_xor_sync(0xffffffffu, g1, 16);
      double kk = h8 ? k1 : k0;
      const double gg = h8 ? k0 : k1;
      kk += __shfl_xor_sync(0xffffffffu, gg, 8);
#pragma unroll
      for (int off = 4; off > 0; off >>= 1) kk += __shfl_xor_sync(0xffffffffu, kk, off);
      if ((lane & 7) == 0) red[warp][(h16 ? 2 : 0) + (h8 ? 1 : 0)] = kk;
    } else {
#pragma unroll
      for (int c = 0; c < KC; ++c) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], off);
      }
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < KC; ++c) red[warp][c] = acc[c];
      }
    }
    __syncthreads();
    if (tid < KC && col0 + tid < ncols) {
      double sum = red[0][tid];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) sum += red[w][tid];
      partial[s * pstride + col0 + tid] = sum;
    }
  }
}

template <int VEC, int MODE, int ALOAD, bool VCOH = false, int KC = kCols, bool FENCE = false>
__device__ __forceinline__ void sweep_tiles(const double* __restrict__ A, long long lda,
                                            long long m, long long ncols,
                                            const double* __restrict__ v,
                                            double* __restrict__ partial, long long pstride,
                                            long long tile_begin, long long tile_stride,
                                            double (*red)[kCols], unsigned& nonfinite,
                                            unsigned& nonzero) {
  const long long S = (m + kChunk - 1) / kChunk;
  const long long G = (ncols + KC - 1) / KC;
  const long long ntiles = S * G;
  for (long long tile = tile_begin; tile < ntiles; tile += tile_stride) {
    const long long s = tile / G;
    const long long g = tile - s * G;
    sweep_tile<VEC, MODE, ALOAD, VCOH, KC, FENCE>(A, lda, m, ncols, v, partial, pstride, s, g, red,
                                                  nonfinite, nonzero);
    __syncthreads();
  }
}

template <int VEC, int MODE, bool STREAM>
__global__ void __launch_bounds__(kThreads, 2) k_sweep(SweepArgs a) {
  if (gate_skip(a.st, a.gate)) return;
  const long long ncols = a.csel ? a.st->d : a.ncols;
  const double* v = a.vsel ? a.vbase + a.st->d * a.vstride : a.v;
  __shared__ double red[kWarps][kCols];
  unsigned nonfinite = 0, nonzero = 0;
  sweep_tiles<VEC, MODE, STREAM ? LOAD_STREAM : LOAD_NC>(a.A, a.lda, a.m, ncols, v, a.partial,
                                                          a.pstride, blockIdx.x, gridDim.x, red,
                                                          nonfinite, nonzero);
  const int tid = threadIdx.x;
  if constexpr (MODE == MODE_INIT) {
    const int any_nf = __syncthreads_or(nonfinite);
    const int any_nz = __syncthreads_or(nonzero);
    if (tid == 0) {
      if (any_nf) atomicOr(&a.st->flags_nonfinite, 1u);
      if (any_nz) atomicOr(&a.st->flags_nonzero, 1u);
    }
  }
}

// ---------------------------------------------------------------------------
// fp32 storage mode of X (rbd_decompose_*_f32): the matrix is held in fp32
// (half the HBM bytes per step), every product and sum is fp64 on the exact
// fp64 value of each element, so the arithmetic is the fp64 path's on the
// fp32-valued matrix. Same tiles (kChunk rows x kCols columns) and partial
// layout as sweep_tiles; a thread owns rows e..e+3, e = 4*(tid + u*kThreads),
// read as one float4 per column when the group is in range and the column
// start is 16-byte aligned (vec4), else as four predicated scalars — the fma
// order is the same either way, so the bits are too.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float4 ld_stream4f(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ bool is_nonfinite_f(float x) {
  return (__float_as_uint(x) & 0x7f800000u) == 0x7f800000u;
}

// KC = columns per tile: 4 (K1) or 8 (the greedy loop: 128 KB per tile, the
// fp64 tile's bytes, loaded as two batches of 16 float4 per thread — row
// groups 0-1 then 2-3 — so per-tile costs are amortised as in fp64). A
// column's sum does not depend on KC.
// Warp + CTA column reduction of sweep_tiles_f32 (KC = 4 or 8): the xor
// butterfly (16, 8, 4, 2, 1) transposed as in sweep_tile: at xor 16 a lane
// keeps half of the columns and receives its partner's copies of them, at
// xor 8 a quarter, ..., down to one column, then xor 2/1 on it. Every sum has
// the butterfly's operands in its order (mine + partner), so the values are
// the plain butterfly's bit for bit, with 9 shuffles per warp for 8 columns
// instead of 40 (4 columns: 6 instead of 20). Lanes (lane & (32/KC - 1)) == 0
// write red[warp][column].
template <int KC>
__device__ __forceinline__ void warp_cols_to_red(const double (&acc)[KC], double (*red)[KC],
                                                 int lane, int warp) {
  static_assert(KC == 4 || KC == 8, "transposed butterfly: 4 or 8 columns");
  const bool h16 = (lane & 16) != 0, h8 = (lane & 8) != 0;
  double k4[KC / 2];
#pragma unroll
  for (int i = 0; i < KC / 2; ++i) {
    const double send = h16 ? acc[i] : acc[KC / 2 + i];
    k4[i] = (h16 ? acc[KC / 2 + i] : acc[i]) + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  double k2[KC / 4];
#pragma unroll
  for (int i = 0; i < KC / 4; ++i) {
    const double send = h8 ? k4[i] : k4[KC / 4 + i];
    k2[i] = (h8 ? k4[KC / 4 + i] : k4[i]) + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double q;
  int col;
  if constexpr (KC == 8) {
    const bool h4 = (lane & 4) != 0;
    const double send = h4 ? k2[0] : k2[1];
    q = (h4 ? k2[1] : k2[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
    q += __shfl_xor_sync(0xffffffffu, q, 2);
    q += __shfl_xor_sync(0xffffffffu, q, 1);
    col = (h16 ? 4 : 0) + (h8 ? 2 : 0) + (h4 ? 1 : 0);
    if ((lane & 3) == 0) red[warp][col] = q;
  } else {
    q = k2[0];
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) q += __shfl_xor_sync(0xffffffffu, q, off);
    col = (h16 ? 2 : 0) + (h8 ? 1 : 0);
    if ((lane & 7) == 0) red[warp][col] = q;
  }
}

// TRAIL = false: no barrier after the partials are written (single-tile calls
// from the persistent loop, whose claim barrier orders `red` for the next
// tile; the caller adds one where a finalisation may read these partials).
template <int MODE, bool VCOH = false, int KC = kCols, bool TRAIL = true>
__device__ __forceinline__ void sweep_tiles_f32(const float* __restrict__ A, long long lda,
                                                long long m, long long ncols,
                                                const double* __restrict__ v,
                                                double* __restrict__ partial, long long pstride,
                                                long long tile_begin, long long tile_stride,
                                                double (*red)[KC], unsigned& nonfinite,
                                                unsigned& nonzero, bool vec4) {
  constexpr int U = kChunk / (4 * kThreads);   // row groups of 4 per thread per column
  constexpr int UB = 16 / KC;                  // row groups per load batch (16 float4 in flight)
  static_assert(U % UB == 0, "batches");
  const long long S = (m + kChunk - 1) / kChunk;
  const long long G = (ncols + KC - 1) / KC;
  const long long ntiles = S * G;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  for (long long tile = tile_begin; tile < ntiles; tile += tile_stride) {
    const long long s = tile / G;
    const long long g = tile - s * G;
    const long long row0 = s * kChunk;
    const long long col0 = g * KC;
    const long long rows = (m - row0 < kChunk) ? m - row0 : kChunk;
    double acc[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) acc[c] = 0.0;
    const float* Ac[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      const long long cc = (col0 + c < ncols) ? col0 + c : col0;  // clamp (result unused)
      Ac[c] = A + cc * lda + row0;
    }
    const double* vr = (MODE == MODE_DOT) ? v + row0 : nullptr;
    auto accum = [&](int c, float4 x, double2 y0, double2 y1) {
      if constexpr (MODE == MODE_DOT) {
        acc[c] = fma((double)x.x, y0.x, acc[c]);
        acc[c] = fma((double)x.y, y0.y, acc[c]);
        acc[c] = fma((double)x.z, y1.x, acc[c]);
        acc[c] = fma((double)x.w, y1.y, acc[c]);
      } else {
        acc[c] = fma((double)x.x, (double)x.x, acc[c]);
        acc[c] = fma((double)x.y, (double)x.y, acc[c]);
        acc[c] = fma((double)x.z, (double)x.z, acc[c]);
        acc[c] = fma((double)x.w, (double)x.w, acc[c]);
        nonfinite |= is_nonfinite_f(x.x) | is_nonfinite_f(x.y) | is_nonfinite_f(x.z) |
                     is_nonfinite_f(x.w);
        nonzero |= (x.x != 0.f) | (x.y != 0.f) | (x.z != 0.f) | (x.w != 0.f);
      }
    };
    auto ldv = [&](const double* p) {
      return VCOH ? __ldcg(reinterpret_cast<const double2*>(p)) : ld_keep2(p);
    };
    if (vec4 && rows == kChunk && col0 + KC <= ncols && lda <= (1LL << 27)) {
      // whole tile in range: batches of UB row groups x KC columns in flight;
      // one base pointer and 32-bit column offsets (fewer live registers)
      // per-column base pointers, element groups at immediate offsets (as in
      // the fp64 sweep: no per-load address arithmetic)
      const float* A0 = A + col0 * lda + row0 + 4 * tid;
      const double* V0 = (MODE == MODE_DOT) ? vr + 4 * tid : nullptr;
#pragma unroll
      for (int ub = 0; ub < U; ub += UB) {
        float4 xv[UB][KC];
        double2 y0[UB], y1[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int eo = (ub + u) * kThreads * 4;
          if constexpr (MODE == MODE_DOT) {
            y0[u] = ldv(V0 + eo);
            y1[u] = ldv(V0 + eo + 2);
          } else {
            y0[u] = y1[u] = make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int c = 0; c < KC; ++c) xv[u][c] = ld_stream4f(A0 + c * lda + eo);
        }
#pragma unroll
        for (int u = 0; u < UB; ++u)
#pragma unroll
          for (int c = 0; c < KC; ++c) accum(c, xv[u][c], y0[u], y1[u]);
      }
    } else {
#pragma unroll 1
      for (int u = 0; u < U; ++u) {
        const long long e = (long long)(tid + u * kThreads) * 4;
        if (e >= rows) break;   // rows past e contribute +0 (a no-op on every sum)
        double2 y0 = make_double2(0.0, 0.0), y1 = make_double2(0.0, 0.0);
        float4 x[KC];
        if (vec4 && e + 4 <= rows) {
          if constexpr (MODE == MODE_DOT) {
            y0 = ldv(vr + e);
            y1 = ldv(vr + e + 2);
          }
#pragma unroll
          for (int c = 0; c < KC; ++c) x[c] = ld_stream4f(Ac[c] + e);
        } else {
          if constexpr (MODE == MODE_DOT) {
            y0.x = __ldcg(vr + e);
            y0.y = (e + 1 < rows) ? __ldcg(vr + e + 1) : 0.0;
            y1.x = (e + 2 < rows) ? __ldcg(vr + e + 2) : 0.0;
            y1.y = (e + 3 < rows) ? __ldcg(vr + e + 3) : 0.0;
          }
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            x[c].x = __ldcg(Ac[c] + e);
            x[c].y = (e + 1 < rows) ? __ldcg(Ac[c] + e + 1) : 0.f;
            x[c].z = (e + 2 < rows) ? __ldcg(Ac[c] + e + 2) : 0.f;
            x[c].w = (e + 3 < rows) ? __ldcg(Ac[c] + e + 3) : 0.f;
          }
        }
#pragma unroll
        for (int c = 0; c < KC; ++c) accum(c, x[c], y0, y1);
      }
    }
    // CTA reduction in a fixed order: xor-butterfly in the warp, then warps 0..7.
    warp_cols_to_red<KC>(acc, red, lane, warp);
    __syncthreads();
    if (tid < KC && col0 + tid < ncols) {
      double sum = red[0][tid];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) sum += red[w][tid];
      partial[s * pstride + col0 + tid] = sum;
    }
    if constexpr (TRAIL) __syncthreads();
  }
}

// K1 over an fp32 matrix (col_sq in fp64, finite / nonzero flags).
static __global__ void __launch_bounds__(kThreads, 2)
    k_sweep_init_f32(const float* __restrict__ A, long long lda, long long m, long long n,
                     double* __restrict__ partial, DevState* st, int vec4) {
  __shared__ double red[kWarps][kCols];
  unsigned nonfinite = 0, nonzero = 0;
  sweep_tiles_f32<MODE_INIT>(A, lda, m, n, nullptr, partial, n, blockIdx.x, gridDim.x, red,
                             nonfinite, nonzero, vec4 != 0);
  const int any_nf = __syncthreads_or(nonfinite);
  const int any_nz = __syncthreads_or(nonzero);
  if (threadIdx.x == 0) {
    if (any_nf) atomicOr(&st->flags_nonfinite, 1u);
    if (any_nz) atomicOr(&st->flags_nonzero, 1u);
  }
}

// ---------------------------------------------------------------------------
// Block-level helpers
// ---------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ double block_sum_fixed(double x, double* sm) {
  // deterministic: xor-butterfly per warp, then warps in order
  for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sm[warp] = x;
  __syncthreads();
  double s = sm[0];
#pragma unroll
  for (int w = 1; w < NT / 32; ++w) s += sm[w];
  __syncthreads();
  return s;
}

// ||w||^2 of the twice-orthogonalised column, w = w1 - Y p. The loops take
// it as ||w1||^2 - ||p||^2 (exact algebra for p = Y'w1 with orthonormal Y),
// which carries ~eps (||w1||^2 + ||p||^2) of rounding. Where that uncertainty
// straddles the breakdown tolerance (decompose.cpp:29-30), the decision is
// made on the norm of the materialised w instead, as the reference does.
__device__ __forceinline__ bool wnorm_in_guard_band(double wn2, double w1n2, double pn, double tol) {
  const double err = 64.0 * 2.220446049250313e-16 * (w1n2 + pn);
  return fabs(wn2 - tol * tol) <= err;
}

// Single-CTA ||w1 - Y p||^2 over all m rows (fixed order: rows strided by the
// CTA's threads, basis vectors in order, then block_sum_fixed). Y, w1 and p
// were written by other CTAs of the grid and are read through L2.
template <int NT>
__device__ __noinline__ double exact_wnorm2(const double* w1, const double* Y, long long m,
                                            long long ldy, long long k, const double* p,
                                            double* sm) {
  double acc = 0.0;
  for (long long i = threadIdx.x; i < m; i += NT) {
    double v = __ldcg(&w1[i]);
    for (long long l = 0; l < k; ++l) v = fma(-__ldcg(&Y[i + l * ldy]), __ldcg(&p[l]), v);
    acc = fma(v, v, acc);
  }
  return block_sum_fixed<NT>(acc, sm);
}

__device__ __forceinline__ void warp_argmax(double& v, long long& j) {
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, off);
    const long long oj = __shfl_xor_sync(0xffffffffu, j, off);
    if (rec_better(ov, oj, v, j)) {
      v = ov;
      j = oj;
    }
  }
}

template <int NT>
__device__ __forceinline__ void block_argmax(double& v, long long& j, Rec* sm) {
  warp_argmax(v, j);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sm[warp] = Rec{v, j};
  __syncthreads();
  v = sm[0].v;
  j = sm[0].j;
#pragma unroll
  for (int w = 1; w < NT / 32; ++w)
    if (rec_better(sm[w].v, sm[w].j, v, j)) {
      v = sm[w].v;
      j = sm[w].j;
    }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// K1 finish: col_sq = sum of chunk partials, residual_sq = col_sq, max col_sq.
// ---------------------------------------------------------------------------
static __global__ void k_init_finish(const double* __restrict__ partial, long long S, long long n,
                              double* __restrict__ col_sq, double* __restrict__ resid,
                              DevState* st) {
  __shared__ double sm[kWarps];
  double mx = 0.0;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (long long s = 0; s < S; ++s) t += partial[s * n + j];
    t = t > 0.0 ? t : 0.0;  // workspace.cpp:37 cwiseMax(0); NaN stays NaN-free only if finite
    col_sq[j] = t;
    resid[j] = t;
    if (t == t && t > mx) mx = t;
  }
  // max is order independent; publish as ordered bits (values >= 0)
  for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = sm[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) b = fmax(b, sm[w]);
    atomicMax(&st->max_colsq_bits, (unsigned long long)__double_as_longlong(b));
  }
}

// ---------------------------------------------------------------------------
// K3: finalize one greedy step.
//   t_j = sum_s partial[s*n + j]      (fixed order: chunk 0..S-1)
//   T[k*n + j] = t_j                  (decompose.cpp:93)
//   r_j = max(r_j - t_j^2, 0)         (workspace.cpp:52-53)
//   argmax over r (value desc, index asc), E_cur = sqrt(max(best, 0))
// mode 0: full decompose step (state update in the last CTA)
// mode 1: workspace extend only (no argmax)
// mode 2: multi-GPU step: local record -> rec_out, no state update
// ---------------------------------------------------------------------------
struct FinalizeArgs {
  const double* partial;
  long long S;
  long long n;
  double* T;            // row-major, row stride n
  long long krow;       // row index (mode 1); modes 0/2 use st->d
  double* r;
  const double* col_sq;
  DevState* st;
  Rec* rec;             // per-CTA records (gridDim.x)
  unsigned* counter;    // last-CTA-done counter (self-resetting)
  double* history;      // device history (mode 0)
  double* cbuf;         // next-step coefficients T[0:d, j*] (mode 0)
  Rec* rec_out;         // mode 2: this rank's record
  long long col_offset; // global index of local column 0
  int mode;
};

static __device__ void finalize_state(const FinalizeArgs& a, double best, long long arg) {
  DevState* st = a.st;
  const long long k = st->d;
  const double e_cur = sqrt(best > 0.0 ? best : 0.0);  // workspace.cpp:123
  a.history[k] = e_cur;                                 // decompose.cpp:99
  st->e_cur = e_cur;
  st->d = k + 1;                                        // :96
  st->jstar = arg;                                      // :101
  st->done = !((k + 1) < st->d_max && e_cur > st->eps_R) ? 1 : 0;  // :87
}

__device__ __forceinline__ void finalize_reduce_tail(const FinalizeArgs& a, long long k, double bv,
                                                     long long bj, Rec* smr, int* is_last_s);

static __global__ void __launch_bounds__(kThreads) k_finalize(FinalizeArgs a) {
  if (a.mode != 1 && a.st->done) return;
  __shared__ Rec smr[kWarps];
  __shared__ int is_last;
  const long long n = a.n;
  const long long k = (a.mode == 1) ? a.krow : a.st->d;
  double* Trow = a.T + k * n;
  double bv = -1.0;  // residual_scan starts best at -1 (workspace.cpp:105)
  long long bj = 0x7fffffffffffffffLL;
  for (long long j = blockIdx.x * (long long)kThreads + threadIdx.x; j < n;
       j += (long long)gridDim.x * kThreads) {
    double t = 0.0;
    for (long long s = 0; s < a.S; ++s) t += a.partial[s * n + j];
    Trow[j] = t;
    const double sq = __dmul_rn(t, t);
    double rj = __dsub_rn(a.r[j], sq);
    rj = rj > 0.0 ? rj : 0.0;
    a.r[j] = rj;
    if (rec_better(rj, j, bv, bj)) {
      bv = rj;
      bj = j;
    }
  }
  if (a.mode == 1) return;
  finalize_reduce_tail(a, k, bv, bj, smr, &is_last);
}

// Shared tail of K3 (mode 0/2): the CTA record, the last CTA's global argmax,
// then (mode 0) the state update and the next step's coefficients.
__device__ __forceinline__ void finalize_reduce_tail(const FinalizeArgs& a, long long k, double bv,
                                                     long long bj, Rec* smr, int* is_last_s) {
  int& is_last = *is_last_s;
  const long long n = a.n;
  __threadfence();  // publish this CTA's T/r writes before the done-counter
  block_argmax<kThreads>(bv, bj, smr);
  if (threadIdx.x == 0) {
    a.rec[blockIdx.x] = Rec{bv, bj};
    __threadfence();
    const unsigned prev = atomicAdd(a.counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  bv = -1.0;
  bj = 0x7fffffffffffffffLL;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += kThreads) {
    const Rec rr{__ldcg(&a.rec[b].v), __ldcg(&a.rec[b].j)};
    if (rec_better(rr.v, rr.j, bv, bj)) {
      bv = rr.v;
      bj = rr.j;
    }
  }
  block_argmax<kThreads>(bv, bj, smr);
  if (threadIdx.x == 0) *a.counter = 0u;
  if (a.mode == 2) {
    if (threadIdx.x == 0) a.rec_out[0] = Rec{bv, bj + a.col_offset};
    return;
  }
  // single GPU: state update + gather of the next step's coefficients
  if (threadIdx.x == 0) {
    finalize_state(a, bv, bj);
    a.st->jlocal = bj;
    a.st->xnorm2 = a.col_sq[bj];
  }
  __syncthreads();
  if (!a.st->done) {
    for (long long l = threadIdx.x; l <= k; l += kThreads) a.cbuf[l] = __ldcg(&a.T[l * n + bj]);
  }
}

// ---------------------------------------------------------------------------
// K4: extension.  w = x - B c (pass 1) / w = w - B p (pass 2), B = Y[:, 0:k].
// CTA = 64 rows x 4 coefficient splits; per-row order fixed (split s takes
// l = s, s+4, ...; the 4 split sums are combined ((s0+s1)+(s2+s3))).
// Each CTA writes sum_rows w^2 to nrm_part[blockIdx.x].
// ---------------------------------------------------------------------------
struct ExtArgs {
  const double* B;      // basis (Y), ld ldb
  long long ldb;
  long long m;
  const double* X;      // pass 1 source: x = X + st->jlocal*ldx (if X != nullptr)
  long long ldx;
  const double* v;      // pass 1 source otherwise (may alias w)
  const double* c;      // coefficients (length k)
  double* w;            // m scratch
  double* nrm_part;     // one per CTA
  DevState* st;
  int gate;
  int pass;             // 1 or 2
};

static __global__ void __launch_bounds__(kThreads) k_ext_gemv_n(ExtArgs a) {
  if (gate_skip(a.st, a.gate)) return;
  const long long k = a.st->d;
  const long long m = a.m;
  __shared__ double cs[kCoefTile];
  __shared__ double part[kGemvSplit][kGemvRows];
  __shared__ double sm[kWarps];
  const int r = threadIdx.x % kGemvRows;
  const int sp = threadIdx.x / kGemvRows;
  const long long i = (long long)blockIdx.x * kGemvRows + r;
  const bool valid = i < m;
  double acc = 0.0;
  for (long long l0 = 0; l0 < k; l0 += kCoefTile) {
    const int nl = (int)((k - l0) < kCoefTile ? (k - l0) : kCoefTile);
    __syncthreads();
    for (int t = threadIdx.x; t < nl; t += kThreads) cs[t] = a.c[l0 + t];
    __syncthreads();
    if (valid) {
      const double* Bp = a.B + i + (l0 + sp) * a.ldb;
      const long long step = (long long)kGemvSplit * a.ldb;
      int l = sp;
      // 8 independent loads in flight per thread
      for (; l + 7 * kGemvSplit < nl; l += 8 * kGemvSplit) {
        double yv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) yv[q] = ld_keep1(Bp + q * step);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = fma(yv[q], cs[l + q * kGemvSplit], acc);
        Bp += 8 * step;
      }
      for (; l < nl; l += kGemvSplit) {
        acc = fma(ld_keep1(Bp), cs[l], acc);
        Bp += step;
      }
    }
  }
  part[sp][r] = acc;
  __syncthreads();
  double wsq = 0.0;
  if (threadIdx.x < kGemvRows) {
    if (valid) {
      const double proj = (part[0][r] + part[1][r]) + (part[2][r] + part[3][r]);
      double x;
      if (a.pass == 1 && a.X != nullptr)
        x = a.X[a.st->jlocal * a.ldx + i];
      else if (a.pass == 1)
        x = a.v[i];
      else
        x = a.w[i];
      const double wi = x - proj;
      a.w[i] = wi;
      wsq = wi * wi;
    }
  }
  const double s = block_sum_fixed<kThreads>(threadIdx.x < kGemvRows ? wsq : 0.0, sm);
  if (threadIdx.x == 0) a.nrm_part[blockIdx.x] = s;
}

// Deterministic single-CTA sum of nparts values.
__device__ __forceinline__ double sum_parts(const double* p, long long np, double* sm) {
  double s = 0.0;
  for (long long b = threadIdx.x; b < np; b += kThreads) s += p[b];
  return block_sum_fixed<kThreads>(s, sm);
}

// After pass 1: decide the second pass exactly as decompose.cpp:28 does.
static __global__ void __launch_bounds__(kThreads) k_ext_decide(const double* nrm_part, long long np,
                                                         DevState* st) {
  if (st->done) return;
  __shared__ double sm[kWarps];
  const double w1n2 = sum_parts(nrm_part, np, sm);
  if (threadIdx.x == 0) {
    st->w1n2 = w1n2;
    const double entry_norm = sqrt(st->xnorm2);
    st->reorth = (st->d > 0) && (st->cfg_reorth || sqrt(w1n2) < 0.5 * entry_norm) ? 1 : 0;
  }
}

// Second-pass coefficients p[l] = sum_s partial[s*pstride + l] (fixed order).
static __global__ void k_coef_combine(const double* __restrict__ partial, long long S, long long pstride,
                               double* __restrict__ p, DevState* st, int gate) {
  if (gate_skip(st, gate)) return;
  const long long k = st->d;
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < k;
       l += (long long)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (long long s = 0; s < S; ++s) t += partial[s * pstride + l];
    p[l] = t;
  }
}

// Norm + breakdown test (decompose.cpp:29-30); on success record selected.
static __global__ void __launch_bounds__(kThreads) k_ext_finish(const double* nrm_part, long long np,
                                                         DevState* st, long long* selected) {
  if (st->done) return;
  __shared__ double sm[kWarps];
  const int re = st->reorth;
  const double wn2 = re ? sum_parts(nrm_part, np, sm) : st->w1n2;
  if (threadIdx.x == 0) {
    const double norm = sqrt(wn2);
    st->wnorm = norm;
    if (norm < st->breakdown_tol || norm == 0.0) {
      st->done = 1;
      st->breakdown = 1;
    } else if (selected != nullptr) {
      selected[st->d] = st->jstar;  // decompose.cpp:94
    }
  }
}

// y = w / norm into the output column (decompose.cpp:31,92).
static __global__ void k_normalize(const double* __restrict__ w, double* __restrict__ ybase,
                            long long ystride, long long m, DevState* st, int use_d) {
  if (st->done) return;
  const double norm = st->wnorm;
  double* y = ybase + (use_d ? st->d * ystride : 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = w[i] / norm;
}

// Entry norm for standalone mgs_project: xnorm2 = ||v||^2 (fixed order).
static __global__ void __launch_bounds__(kThreads) k_norm2_single(const double* v, long long m,
                                                           DevState* st) {
  __shared__ double sm[kWarps];
  double s = 0.0;
  for (long long i = threadIdx.x; i < m; i += kThreads) s = fma(v[i], v[i], s);
  s = block_sum_fixed<kThreads>(s, sm);
  if (threadIdx.x == 0) st->xnorm2 = s;
}

// Workspace scan (residual_scan identity, workspace.cpp:101-125) into out.
static __global__ void __launch_bounds__(kThreads) k_scan_only(const double* r, long long n, Rec* rec,
                                                        unsigned* counter, Rec* out) {
  __shared__ Rec smr[kWarps];
  __shared__ int is_last;
  double bv = -1.0;
  long long bj = 0x7fffffffffffffffLL;
  for (long long j = blockIdx.x * (long long)kThreads + threadIdx.x; j < n;
       j += (long long)gridDim.x * kThreads)
    if (rec_better(r[j], j, bv, bj)) {
      bv = r[j];
      bj = j;
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

// Identity error_sq (workspace.cpp:84-99) for one column from the T rows.
static __global__ void k_error_sq(const double* T, long long n, long long d, long long j,
                           const double* c, const double* col_sq, double* out) {
  __shared__ double sm[kWarps];
  double cross = 0.0, quad = 0.0;
  for (long long k = threadIdx.x; k < d; k += kThreads) {
    cross = fma(c[k], T[k * n + j], cross);
    quad = fma(c[k], c[k], quad);
  }
  cross = block_sum_fixed<kThreads>(cross, sm);
  quad = block_sum_fixed<kThreads>(quad, sm);
  if (threadIdx.x == 0) {
    const double e2 = col_sq[j] - 2.0 * cross + quad;
    out[0] = e2 > 0.0 ? e2 : 0.0;
  }
}

}  // namespace rbdk

namespace rbdk {

// ===========================================================================
// Fused extension (decompose loop). Y is read from HBM once per step.
//
// Step k (k = st->d accepted columns; column k-1 may be "pending": its
// second-pass correction not yet applied). For every 32-row block:
//   phase 1 (one HBM read of Y[rows, 0:kb], kb = materialised columns):
//     y_{k-1}  = (w1_{k-1} - Y p_{k-1}) / ||w_{k-1}||   -> Y[:, k-1]
//     w1_k     = x_{j*} - Y[:, 0:k] c,   c = T[0:k, j*]  (CGS pass 1)
//   phase 2 (re-read of the same block, L2 resident):
//     p_k     += Y[rows, 0:k]' w1_k[rows]                (reorth coefficients)
// k_ext_reduce then sums the CTA partials, applies decompose.cpp:28's
// condition (second pass iff reorthogonalize or ||w1|| < 0.5 ||x||), sets
// ||w_k||^2 = ||w1||^2 - ||p||^2 and performs the breakdown test (:29-30).
// The sweep runs on the unnormalised w1_k and k_finalize_fused forms
//   T[k, j] = (w1_k . x_j - p_k . T[0:k, j]) / ||w_k||  ( = y_k . x_j ).
// ===========================================================================
constexpr int kFRows = 32;        // rows per fused-extension block
constexpr int kFMaxCoef = 4096;   // fused path handles d_max <= this

struct FusedArgs {
  double* Y;              // m x d_max column-major (ld m)
  long long m;
  const double* X;        // x = X + st->jlocal * ldx (if X != nullptr)
  long long ldx;
  const double* xsrc;     // otherwise x = xsrc
  const double* c;        // T[0:k, j*]
  const double* p;        // p_{k-1} (zeroed when the pass was skipped)
  double* w;              // in: w1_{k-1}; out: w1_k
  double* ppart;          // [gridDim.x][pstride]
  long long pstride;
  double* npart;          // [gridDim.x]
  DevState* st;
  long long dcap;         // coefficient capacity (= d_max) of the smem arrays
};

static __global__ void __launch_bounds__(kThreads) k_ext_fused(FusedArgs a) {
  DevState* st = a.st;
  const int pending = st->pending;
  const int live = !st->done;
  if (!pending && !live) return;
  const long long k = st->d;
  const long long kb = pending ? k - 1 : k;  // columns already materialised
  const long long m = a.m;
  extern __shared__ double fsm[];
  double* cs = fsm;                 // c[0:k]
  double* ps = cs + a.dcap;         // p_{k-1}[0:kb]
  double* pacc = ps + a.dcap;       // this CTA's p_k partial [0:k]
  __shared__ double red_c[kWarps][kFRows];
  __shared__ double red_p[kWarps][kFRows];
  __shared__ double w1s[kFRows];
  __shared__ double yns[kFRows];
  __shared__ double smn[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (long long l = tid; l < k; l += kThreads) {
    cs[l] = live ? a.c[l] : 0.0;
    pacc[l] = 0.0;
  }
  for (long long l = tid; l < kb; l += kThreads) ps[l] = pending ? a.p[l] : 0.0;
  const double wprev_norm = st->wnorm;
  const double* x = a.X ? a.X + st->jlocal * a.ldx : a.xsrc;
  __syncthreads();

  const long long nblk = (m + kFRows - 1) / kFRows;
  const long long b0 = nblk * blockIdx.x / gridDim.x;
  const long long b1 = nblk * (blockIdx.x + 1) / gridDim.x;
  double nacc = 0.0;
  for (long long b = b0; b < b1; ++b) {
    const long long row0 = b * kFRows;
    // ---- phase 1: lane = row, warp w takes l = w, w+8, ... ----
    {
      const long long i = row0 + lane;
      const bool ok = i < m;
      double acc_c = 0.0, acc_p = 0.0;
      if (ok) {
        const double* yp = a.Y + i + (long long)warp * m;
        const long long stp = (long long)kWarps * m;
        long long l = warp;
        for (; l + 7 * kWarps < kb; l += 8 * kWarps) {
          double yv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) yv[q] = yp[q * stp];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            acc_c = fma(yv[q], cs[l + q * kWarps], acc_c);
            acc_p = fma(yv[q], ps[l + q * kWarps], acc_p);
          }
          yp += 8 * stp;
        }
        for (; l < kb; l += kWarps) {
          const double y0 = *yp;
          acc_c = fma(y0, cs[l], acc_c);
          acc_p = fma(y0, ps[l], acc_p);
          yp += stp;
        }
      }
      red_c[warp][lane] = acc_c;
      red_p[warp][lane] = acc_p;
      __syncthreads();
      if (warp == 0) {
        double sc = red_c[0][lane], sp = red_p[0][lane];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) {
          sc += red_c[w][lane];
          sp += red_p[w][lane];
        }
        double yk1 = 0.0, w1 = 0.0;
        if (ok) {
          if (pending) {
            yk1 = (a.w[i] - sp) / wprev_norm;        // second pass of column k-1
            a.Y[i + (k - 1) * m] = yk1;
            sc = fma(yk1, cs[k - 1], sc);
          }
          if (live) {
            w1 = x[i] - sc;                          // first pass of column k
            a.w[i] = w1;
            nacc = fma(w1, w1, nacc);
          }
        }
        w1s[lane] = w1;
        yns[lane] = yk1;
      }
      __syncthreads();
    }
    if (!live) continue;
    // ---- phase 2: p_k += Y[rows, 0:k]' w1 (lane = 8 columns x 4 row segments) ----
    {
      const int cq = lane >> 2, rs = lane & 3;
      double wv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) wv[q] = w1s[rs * 8 + q];
      const long long ib = row0 + rs * 8;
      const int nrow = (int)((m - ib) < 8 ? (m - ib) : 8);
      // warp-uniform trip count: every lane reaches the shuffles
      for (long long lb = warp * 8; lb < kb; lb += 64) {
        const long long l = lb + cq;
        double s = 0.0;
        if (l < kb) {
          const double* yp = a.Y + ib + l * m;
          if (nrow == 8) {
#pragma unroll
            for (int q = 0; q < 8; ++q) s = fma(yp[q], wv[q], s);
          } else {
            for (int q = 0; q < nrow; ++q) s = fma(yp[q], wv[q], s);
          }
        }
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (rs == 0 && l < kb) pacc[l] += s;
      }
      if (pending && warp == 0) {   // the column materialised in phase 1
        double s = yns[lane] * w1s[lane];
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) pacc[k - 1] += s;
      }
    }
    __syncthreads();
  }
  // publish the CTA partials
  if (live) {
    for (long long l = tid; l < k; l += kThreads) a.ppart[blockIdx.x * a.pstride + l] = pacc[l];
    const double s = block_sum_fixed<kThreads>(warp == 0 ? nacc : 0.0, smn);
    if (tid == 0) a.npart[blockIdx.x] = s;
  }
}

// Sum of the k_ext_fused partials, the reorth decision, ||w_k|| and the
// breakdown test. Grid: ceil(k/32) CTAs of 256 threads (32 columns x 8 splits)
// plus a last-CTA finish.
struct ReduceArgs {
  const double* ppart;
  long long pstride;
  int nparts;
  const double* npart;
  double* p;              // out: p_k (zeroed if the second pass is skipped)
  DevState* st;
  long long* selected;
  const double* w1;       // w1 (m), for the guard-band norm recompute
  const double* Y;        // m x k basis, ld m
  long long m;
};

static __global__ void __launch_bounds__(kThreads) k_ext_reduce(ReduceArgs a) {
  DevState* st = a.st;
  __shared__ double sred[kWarps][32];
  __shared__ double smn[kWarps];
  __shared__ int is_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int live = !st->done;
  const long long k = st->d;
  if (live) {
    const long long l = (long long)blockIdx.x * 32 + lane;
    double s = 0.0;
    if (l < k)
      for (int b = warp; b < a.nparts; b += kWarps) s += a.ppart[(long long)b * a.pstride + l];
    sred[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && l < k) {
      double t = sred[0][lane];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) t += sred[w][lane];
      a.p[l] = t;
    }
    __threadfence();
  }
  __syncthreads();
  if (tid == 0) is_last = (atomicAdd(&st->counter_b, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (tid == 0) st->counter_b = 0u;
  const int pending_was = st->pending;
  if (!live) {
    if (tid == 0 && pending_was) st->pending = 0;   // materialised by k_ext_fused
    return;
  }
  double w1n2 = 0.0;
  for (int b = tid; b < a.nparts; b += kThreads) w1n2 += a.npart[b];
  w1n2 = block_sum_fixed<kThreads>(w1n2, smn);
  double pn = 0.0;
  for (long long l = tid; l < k; l += kThreads) {
    const double v = __ldcg(&a.p[l]);
    pn = fma(v, v, pn);
  }
  pn = block_sum_fixed<kThreads>(pn, smn);
  const int reorth = (k > 0) && (st->cfg_reorth || sqrt(w1n2) < 0.5 * sqrt(st->xnorm2));
  double wn2 = reorth ? w1n2 - pn : w1n2;
  if (reorth && wnorm_in_guard_band(wn2, w1n2, pn, st->breakdown_tol))
    wn2 = exact_wnorm2<kThreads>(a.w1, a.Y, a.m, a.m, k, a.p, smn);
  __syncthreads();
  if (!reorth)
    for (long long l = tid; l < k; l += kThreads) a.p[l] = 0.0;
  if (tid == 0) {
    st->pending = 0;
    st->reorth = reorth;
    st->w1n2 = w1n2;
    wn2 = wn2 > 0.0 ? wn2 : 0.0;
    const double norm = sqrt(wn2);
    if (norm < st->breakdown_tol || norm == 0.0) {
      st->done = 1;
      st->breakdown = 1;
    } else {
      st->wnorm = norm;
      if (a.selected) a.selected[k] = st->jstar;
    }
  }
}

// K3 for the fused path: combine sweep partials, apply the reorth correction
// and the normalisation, update residuals, argmax, state.
struct Finalize2Args {
  const double* partial;
  long long S;
  long long n;
  double* T;
  const double* p;
  double* r;
  const double* col_sq;
  DevState* st;
  Rec* rec;
  unsigned* counter;
  double* history;
  double* cbuf;
  Rec* rec_out;          // multi-GPU: local record, no state update
  long long col_offset;
  int mode;              // 0 single GPU, 2 multi-GPU local
};

constexpr int kF2Cols = 32;   // columns per CTA
static __global__ void __launch_bounds__(kThreads) k_finalize_fused(Finalize2Args a) {
  DevState* st = a.st;
  if (st->done) return;
  __shared__ double scorr[kWarps][kF2Cols];
  __shared__ Rec smr[kWarps];
  __shared__ int is_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long n = a.n;
  const long long k = st->d;
  const double norm = st->wnorm;
  const int reorth = st->reorth;
  double* Trow = a.T + k * n;
  double bv = -1.0;
  long long bj = 0x7fffffffffffffffLL;
  const long long ngroups = (n + kF2Cols - 1) / kF2Cols;
  for (long long g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const long long j = g * kF2Cols + lane;
    const bool ok = j < n;
    // correction p . T[0:k, j], l split over the 8 warps
    double corr = 0.0;
    if (ok && reorth) {
      for (long long l = warp; l < k; l += kWarps) corr = fma(a.p[l], a.T[l * n + j], corr);
    }
    scorr[warp][lane] = corr;
    // chunk partials (warp w sums chunks s = w, w+8, ... ; combined in order below)
    __syncthreads();
    if (warp == 0) {
      double c = scorr[0][lane];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) c += scorr[w][lane];
      if (ok) {
        double t = 0.0;
        for (long long s = 0; s < a.S; ++s) t += a.partial[s * n + j];
        t = (t - c) / norm;
        Trow[j] = t;
        const double sq = __dmul_rn(t, t);
        double rj = __dsub_rn(a.r[j], sq);
        rj = rj > 0.0 ? rj : 0.0;
        a.r[j] = rj;
        if (rec_better(rj, j, bv, bj)) {
          bv = rj;
          bj = j;
        }
      }
    }
    __syncthreads();
  }
  __threadfence();
  block_argmax<kThreads>(bv, bj, smr);
  if (tid == 0) {
    a.rec[blockIdx.x] = Rec{bv, bj};
    __threadfence();
    is_last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  bv = -1.0;
  bj = 0x7fffffffffffffffLL;
  for (unsigned b = tid; b < gridDim.x; b += kThreads) {
    const Rec rr{__ldcg(&a.rec[b].v), __ldcg(&a.rec[b].j)};
    if (rec_better(rr.v, rr.j, bv, bj)) {
      bv = rr.v;
      bj = rr.j;
    }
  }
  block_argmax<kThreads>(bv, bj, smr);
  if (tid == 0) *a.counter = 0u;
  if (a.mode == 2) {
    if (tid == 0) a.rec_out[0] = Rec{bv, bj + a.col_offset};
    return;
  }
  if (tid == 0) {
    const double e_cur = sqrt(bv > 0.0 ? bv : 0.0);   // workspace.cpp:123
    a.history[k] = e_cur;                              // decompose.cpp:99
    st->e_cur = e_cur;
    st->d = k + 1;                                     // :96
    st->pending = 1;                                   // y_k awaits its second pass
    st->jstar = bj;                                    // :101
    st->jlocal = bj;
    st->xnorm2 = a.col_sq[bj];
    st->done = !((k + 1) < st->d_max && e_cur > st->eps_R) ? 1 : 0;  // :87
  }
  __syncthreads();
  if (!st->done) {
    for (long long l = tid; l <= k; l += kThreads) a.cbuf[l] = __ldcg(&a.T[l * n + bj]);
  }
}

}  // namespace rbdk
