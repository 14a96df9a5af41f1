// rbd_persistent.cuh — the whole RBD greedy loop (decompose.cpp:87-102) as ONE
// persistent cooperative kernel: one CTA pair per SM stays resident for all
// steps; the phases of a step are separated by grid barriers instead of
// kernel launches, and every CTA carries an identical copy of the (tiny) loop
// state, so no host round trip or graph replay happens inside the loop.
//
// Step k (k accepted columns, column k-1 possibly "pending"):
//   P1  extension pass over this CTA's rows (one HBM read of Y):
//         y_{k-1} = (w1_{k-1} - Y p_{k-1}) / ||w_{k-1}||   -> Y[:, k-1]
//         w1_k    = x_{j*} - Y c,   c = T[0:k, j*]           (+ ||w1_k||^2)
//   --- no barrier: each CTA publishes the rows it finished (per 4096-row
//       chunk, release-add); an X tile of chunk s starts once chunk s is
//       complete, the Y'w1 tiles once every CTA is through P1 ---
//   P2  one dynamically scheduled tile queue:
//         Y'w1 tiles (reorth coefficients p_k; Y is still L2-hot) — the last
//           one decides the second pass (decompose.cpp:28), ||w_k|| and the
//           breakdown test (:29-30) and publishes them;
//         X'w1 tiles (the fused sweep) — the last chunk of a 4-column group
//           finalises T[k, j] = (w1_k . x_j - p_k . T[0:k, j]) / ||w_k||, the
//           residuals (workspace.cpp:52-53) and a group record; the last group
//           publishes the global argmax (workspace.cpp:107-113,123).
//   --- barrier ---
//       every CTA: stop test (decompose.cpp:87) on the published outcome
//
// DIAG (diagonal weight A = diag(a), row f1): Y and T stay Euclidean; the scan
// is on e2_j = ||x_j||_A^2 - 2 cross_j + quad_j (rbd_weighted.cuh). With the
// lazy xi_k = (w1 - Y p)/||w||, P1 also writes a o w1 and w1'Aw1, the Y'w1 and
// X tiles take two vectors (w1, a o w1) in the same pass, and
//   YAX[k, j]   = ((a o w1).x_j - p.YAX[0:k, j]) / ||w||
//   YAY[k, 0:k] = (q - YAY p) / ||w||,   q = Y'(a o w1)
//   YAY[k, k]   = (w1'Aw1 - 2 p.q + p'YAY p) / ||w||^2
// (the decider forms the YAY row; the finaliser carries cross/quad).
#pragma once

#include "rbd_select.h"
#include "rbd_weighted.cuh"

namespace rbdk {

struct PersistArgs {
  const double* X;
  const float* Xf;    // XF32 instantiation: X stored in fp32 (arithmetic stays fp64)
  int xvec4;          // XF32: ldx % 4 == 0 and Xf 16-byte aligned (float4 loads)
  long long ldx;
  long long m;
  long long n;
  double* Y;
  double* T;
  double* w;
  double* p;
  double* ppart;      // [G][d_max]
  double* npart;      // [G]
  double* partial;    // [S][n]
  double* r;
  const double* col_sq;
  Rec* rec;           // [G]
  double* history;
  long long* selected;
  DevState* st;
  unsigned* bar;      // [0] arrival count, [1] generation
  long long d_max;
  unsigned long long* phase_ns;  // optional [8] accumulated phase times (CTA 0)
  unsigned long long* trace;     // optional per-CTA timeline [G][kTraceWords] for steps
  long long trace_step;          //   trace_step .. trace_step+1
  // sharded mode (one step per launch; see rbd_shard.cu)
  const double* recv;            // the winner's payload (allreduced: owner's values + -0.0)
  double* send;                  // this rank's 16-byte record {best residual, global index}
  long long pay_stride;          // doubles per payload
  long long col_offset;          // global index of local column 0
  struct StepCtl* ctl;           // queue / publish words
  unsigned long long* rdy;       // [0] CTAs through P1, [1 + s] rows of chunk s written by P1
                                 // (monotonic within a decompose, zeroed with ctl)
  long long* progress;           // optional mapped host word: Y columns [0, value) are final
  // test instrumentation (SURVEY §8(c) parity protocol): steps k < nforced
  // select forced[k] instead of the argmax (history still records the argmax)
  const long long* forced;
  long long nforced;
  // diagonal weight A = diag(a) (DIAG instantiation; see rbd_weighted.cuh)
  const double* diag;            // a
  double* aw;                    // a o w1_k (P1)
  double* npart2;                // [G] P1 shares of w1' A w1
  double* ppart2;                // [S][d_max] chunk partials of Y'(a o w1)
  double* q;                     // [d_max] q_k = Y'(a o w1_k)
  double* partial2;              // [S][n] X-tile partials of (a o w1).x_j (NaN = not written)
  double* YAX;                   // [d_max][n] YAX[l, j] = (A y_l).x_j
  double* YAY;                   // [d_max][d_max] Y'AY (symmetric)
  double* yrow;                  // [d_max + 1] YAY[k, 0:k+1] of the current step
  double* cross;                 // [n] sum_l T[l,j] YAX[l,j]
  double* quad;                  // [n] T[:,j]' YAY T[:,j]
  const double* colsq_a;         // [n] ||x_j||_A^2
  double* yslice;                // [d_max / kYSlice + 2][2] per-slice (p.q, p.v) of the YAY row
  // identity loops: the first ydelay claims of a step are X tiles, then the
  // Y'w1 groups, then the rest (CTAs that claim first then stream X instead
  // of waiting for every CTA's P1; the decision comes a tile later)
  long long ydelay;
  // FOLD instantiation: steps with k <= fold_kmax form p_k = Y'w1_k inside P1
  // (each CTA's share from the row block it just read, re-read from L2) and
  // the Y'w1 groups only sum the G shares; larger k sweep Y as before
  long long fold_kmax;
};

__device__ __forceinline__ void red_release_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ long long ld_acquire_s64_(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void wait_step_ne(const long long* flag, long long bad) {
  const unsigned long long t0 = globaltimer();
  unsigned spins = 0;
  while (ld_acquire_s64_(flag) == bad) {
    __nanosleep(32);
    if ((++spins & 0xfffu) == 0 && globaltimer() - t0 > 30000000000ull) __trap();
  }
}

// Grid barrier (all CTAs co-resident: cooperative launch): one monotonic
// arrival counter, release-add on arrival, acquire-poll until it reaches the
// next multiple of gridDim.x. The counter is zeroed before every decompose
// and every launch of one decompose uses the same grid, so barrier b of the
// call completes at b * gridDim.x. Traps after 30 s instead of hanging.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    const unsigned goal = (old / gridDim.x + 1) * gridDim.x;
    const unsigned long long t0 = globaltimer();
    unsigned spins = 0;
    while ((int)(ld_acquire_u32(bar) - goal) < 0) {
      if ((++spins & 0xffffu) == 0 && globaltimer() - t0 > 30000000000ull) __trap();
    }
    gen = goal;
  }
  __syncthreads();
}

// Shared step bookkeeping (device memory, see PersistArgs::ctl).
struct StepCtl {
  unsigned long long tile_ctr;   // tile-claim counter: 0 at kernel entry, then monotonic
  unsigned ydone;                // Y'w1 groups finished this step (reset by the decider)
  unsigned pad;
  // published by the decider (claimer of the last Y'w1 tile), tagged with step+1
  long long p_step;
  double norm;
  int reorth;
  int breakdown;
  // published by the claimer of the last tile, tagged with step+1
  long long r_step;
  double e_cur;
  long long jstar;
  // DIAG: the YAY row of the step, computed in slices by every CTA after the
  // decision; the CTA finishing the last slice publishes it, tagged step+1
  unsigned yslices;              // CTAs through their slices this step
  unsigned pad3;
  long long y_step;
  double w1a;                    // w1'Aw1 (the decider's sum)
};

__device__ __forceinline__ long long ld_acquire_s64(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_s64(long long* p, long long v) {
  asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// Poll a value produced by an earlier-claimed tile (NaN = not yet written).
__device__ __forceinline__ double poll_f64(const double* p) {
  double v = ld_relaxed_f64(p);
  if (v == v) return v;
  const unsigned long long t0 = globaltimer();
  unsigned spins = 0;
  do {
    __nanosleep(32);
    v = ld_relaxed_f64(p);
    if ((++spins & 0xfffu) == 0 && globaltimer() - t0 > 30000000000ull) __trap();
  } while (v != v);
  return v;
}

__device__ __forceinline__ void wait_step(const long long* flag, long long want) {
  const unsigned long long t0 = globaltimer();
  unsigned spins = 0;
  while (ld_acquire_s64(flag) != want) {
    __nanosleep(32);
    if ((++spins & 0xfffu) == 0 && globaltimer() - t0 > 30000000000ull) __trap();
  }
}

#define kNaN __longlong_as_double(-1LL)

__device__ __forceinline__ bool live_at_exit(int done, int breakdown) {
  return !done && !breakdown;
}

constexpr int kP3Groups = 4;   // column groups finalised together in P3
#ifndef RBD_P1_LOADS
#define RBD_P1_LOADS 16
#endif
constexpr int kPLoads = RBD_P1_LOADS;   // P1: Y loads in flight per lane per batch
constexpr int kYSlice = kWarps;         // DIAG: YAY-row entries per slice (one warp each)
constexpr int kTraceWords = 256;  // per CTA: [0] count, then (tag<<40 | time) words

// Payload of a rank in sharded mode (doubles): [0] best residual, [1] global
// column index (bits), [2] col_sq of that column, [3] pad, [4, 4+m) the
// column x_j, [4+m, 4+m+k+1) the column T[0:k+1, j].
constexpr int kPayHead = 4;

#ifndef RBD_INSTRUMENT
#define RBD_INSTRUMENT 0   // 1: RBD_PHASE_TIMING / RBD_TRACE_STEP work (tools only)
#endif
#ifndef RBD_FOLD_ROWS
#define RBD_FOLD_ROWS 64   // FOLD P1 block height (64: one half of 8 warps; 128: two halves)
#endif
// Columns of p_k summed per Y'w1 group in a FOLD step (the G CTA shares).
constexpr int kFoldCols = 32;

// One level of the FOLD transposing butterfly: S values per lane; the lane
// keeps the half selected by its lane bit BIT and adds the partner's copy of
// that half (one shuffle per kept value).
template <int S, int BIT>
__device__ __forceinline__ void fold_butterfly(double* t, int lane) {
  const bool upper = (lane & BIT) != 0;
#pragma unroll
  for (int q = 0; q < S; ++q) {
    const double send = upper ? t[q] : t[q + S];
    const double keep = upper ? t[q + S] : t[q];
    t[q] = keep + __shfl_xor_sync(0xffffffffu, send, BIT);
  }
}

// FOLD, P1: one row block's share of p_k = Y[:, 0:k]' w1_k, added into psh
// (shared). The block is re-read from L2 (column k-1 was just written by P1);
// a lane holds two rows (yb = Y + its first row; wa, wb their w1), and a
// transposing butterfly leaves lane pair 2c..2c+1 with column c of the
// 16-column batch summed over the half's 64 rows. The most recently read
// batches are re-read first (fewer L2 misses: C2 3058 -> 3055 ms against
// in-order re-reads below k = 448).
template <int PW>
__device__ __forceinline__ void fold_block_share(const double* __restrict__ yb, long long m, long long k,
                                              int wh, int lane, double wa, double wb, bool rows,
                                              double* psh) {
  constexpr int kStep = kPLoads * PW;
  const long long nb = (k - wh + kStep - 1) / kStep;
  for (long long bi = 0; bi < nb; ++bi) {
    const long long l = wh + (nb - 1 - bi) * kStep;
    double t[kPLoads];
#pragma unroll
    for (int q = 0; q < kPLoads; ++q) {
      const long long col = l + q * PW;
      double2 v = make_double2(0.0, 0.0);
      if (rows && col < k) v = __ldcg(reinterpret_cast<const double2*>(yb + col * m));
      t[q] = fma(v.y, wb, v.x * wa);
    }
    fold_butterfly<8, 16>(t, lane);
    fold_butterfly<4, 8>(t, lane);
    fold_butterfly<2, 4>(t, lane);
    fold_butterfly<1, 2>(t, lane);
    t[0] += __shfl_xor_sync(0xffffffffu, t[0], 1);
    const int qs = (((lane >> 4) & 1) << 3) | (((lane >> 3) & 1) << 2) | (((lane >> 2) & 1) << 1) |
                   ((lane >> 1) & 1);
    const long long col = l + qs * PW;
    if ((lane & 1) == 0 && col < k) psh[col] += t[0];   // (warp, lane pair) owns col
  }
}

// FOLD, Y'w1 group t: p_k[l] = sum of the G CTA shares (ppart[b][l]) for
// the group's kFoldCols columns, in a fixed order: 8 strided partial sums per
// column, then the partials in order (rp: kThreads doubles of shared memory).
static __device__ __noinline__ void fold_group_sum(const double* ppart, long long d_max, int G, long long k,
                                            long long t, double* rp, double* pk) {
  constexpr int kParts = kThreads / kFoldCols;
  const int tid = threadIdx.x;
  const int cl = tid % kFoldCols, part = tid / kFoldCols;
  const long long l = t * kFoldCols + cl;
  double v = 0.0;
  if (l < k)
    for (int b = part; b < G; b += kParts) v += __ldcg(&ppart[(long long)b * d_max + l]);
  rp[part * kFoldCols + cl] = v;
  __syncthreads();
  if (tid < kFoldCols && l < k) {
    double sum = rp[cl];
#pragma unroll
    for (int pp = 1; pp < kParts; ++pp) sum += rp[pp * kFoldCols + cl];
    pk[l] = sum;
  }
}

template <int VEC, bool SHARD, bool DIAG = false, bool XF32 = false, bool FOLD = false>
__global__ void __launch_bounds__(kThreads, 2) k_rbd_persistent(PersistArgs a) {
  static_assert(!(SHARD && DIAG), "the weighted loop is single-GPU");
  static_assert(!XF32 || (!SHARD && !DIAG), "fp32 storage: single-GPU identity loop");
  static_assert(!FOLD || (VEC == 2 && !DIAG && !SHARD), "fold: single-GPU identity loop, row pairs");
  // The fold lives in its own instantiation: compiled into the base kernel
  // (runtime-gated) it cost that kernel's X-tile stream 4-9% on C1/C2
  // (ptxas then consumed a batch's first loads before issuing the rest).
  constexpr bool FC = FOLD;
  extern __shared__ __align__(128) double dsm[];
  // P1 block: halves of 32*VEC rows (warps 0-3 / 4-7); within a half the kPW
  // warps split the columns (l = wh mod kPW), so every row's sum runs in the
  // same order whichever half it falls in. FOLD: one 64-row half of all 8
  // warps, so the 296 CTAs' blocks (64 x k doubles each) stay L2-resident
  // until the block's Y'w1 share re-reads them (tools/microbench/p1_fold.cu:
  // 128-row blocks miss L2 at k >= 256)
  constexpr bool kOneHalf = FOLD && RBD_FOLD_ROWS == 64;
  constexpr int kPW = kOneHalf ? kWarps : kWarps / 2;   // warps per half
  constexpr int kPHalf = 32 * VEC;
  constexpr int kPRows = kOneHalf ? kPHalf : 2 * kPHalf;  // rows per P1 block
  constexpr int kNHalf = kPRows / kPHalf;
  constexpr int kPBatch = kPLoads * kPW;   // columns per P1 batch of a half
  static_assert(kPBatch <= 16 * kWarps, "P1 batch padding (persist_smem) too small");
  double* cs = dsm;                        // c = T[0:k, j*], zero-padded to a batch multiple
  double* ps = cs + a.d_max + kPBatch;     // p_{k-1} (pending column), zero-padded
  double* pd = cs + 2 * (a.d_max + kPBatch);    // DIAG: p_k (finaliser copy)
  double* yd = pd + a.d_max + 1;                // DIAG: YAY[k, 0:k+1]
  // DIAG, VEC 2: per-thread cp.async slots of the X tiles' two vectors
  double2* svec = reinterpret_cast<double2*>(cs + ((2 * (a.d_max + 16 * kWarps) + 2 * (a.d_max + 1) + 1) & ~1LL));
  // FOLD: this CTA's share of p_k, per half (recomputed at each use: nothing
  // of the fold stays live across the X-tile queue)
  auto psh = [&] { return dsm + 2 * (a.d_max + 16 * kWarps); };
  __shared__ double red[kWarps][kCols];
  __shared__ double w1s[FC ? kPRows : 1];         // FOLD: w1 of the block's rows
  __shared__ double red_c[kWarps][kPHalf];
  __shared__ double red_p[kWarps][kPHalf];
  __shared__ double smn[kWarps];
  __shared__ Rec smr[kWarps];
  __shared__ long long sh_tile;
  __shared__ int sh_ok;
  __shared__ int sh_dec[2];
  __shared__ double sh_decd[2];
  // DIAG two-vector tiles reduce through red_c (free outside P1)
  double (*red2)[2 * kCols] = reinterpret_cast<double (*)[2 * kCols]>(&red_c[0][0]);
  static_assert(sizeof(red_c) >= sizeof(double) * kWarps * 2 * kCols, "red2 alias");

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long m = a.m, n = a.n;
  const int G = gridDim.x, cta = blockIdx.x;
  DevState* st = a.st;
  StepCtl* ctl = a.ctl;
  unsigned gen = 0;
  if (tid == 0) gen = ld_acquire_u32(&a.bar[1]);
  // the claim counter is 0 at entry (ctl is zeroed before a single-GPU launch;
  // in sharded mode CTA 0 rezeroes it after the step's last barrier), and
  // advances by exactly total + G per step
  unsigned long long tile_base = 0;

  // ---- loop state: identical in every CTA (and, sharded, on every rank) ----
  long long k = st->d;
  // P1 publications are counted from the k the counters were zeroed at
  const long long k_base = SHARD ? 0 : k;
  long long jstar = st->jstar;
  int done = st->done;
  int pending = 0, reorth_prev = 0, breakdown = 0;
  double wnorm_prev = 1.0, e_cur = st->e_cur;
  double xnorm2 = 0.0;
  const double* pay = nullptr;   // sharded: the winner's payload
  if constexpr (SHARD) {
    pending = st->pending;
    reorth_prev = st->reorth;
    wnorm_prev = st->wnorm;
    xnorm2 = st->xnorm2;
    pay = a.recv;
  } else {
    xnorm2 = a.col_sq[jstar];
  }
  const double eps_R = st->eps_R, tol = st->breakdown_tol;
  const int cfg_reorth = st->cfg_reorth;
  // (m, n >= 0: unsigned shifts, cheap to rematerialise in the tile loop)
  const long long S = (long long)((unsigned long long)(m + kChunk - 1) / kChunk);
  // p_k by step parity: a CTA still in P1 of step k reads p_{k-1} while
  // faster CTAs already write p_k
  auto pbuf = [&](long long kk) { return a.p + (kk & 1) * (a.d_max + 1); };
  // P1 row range of this CTA: an even split of the rows (kept even so 16-byte
  // row pairs never straddle two CTAs), processed in kPRows-row blocks
  const long long r_lo = ((m * cta / G) + 1) & ~1LL;
  const long long r_hi = (cta + 1 == G) ? m : (((m * (cta + 1) / G) + 1) & ~1LL);
  const long long ngx = (long long)((unsigned long long)(n + kCols - 1) / kCols);   // X column groups (finalisation unit)
  constexpr int kXT = XF32 ? 2 * kCols : kCols;    // columns per X tile (fp32: 128 KB tiles)
  const long long ngt = (long long)((unsigned long long)(n + kXT - 1) / kXT);       // X tile columns
  const long long nx = ngt * S;                    // X tiles
  const double rS = 1.0 / (double)S;
  // X claim index tx (counted after the Y'w1 groups) -> column group g and
  // chunk s; used for the tile and for its P1-readiness wait. Group-major; DIAG
  // puts every group's last chunk at the end instead (measured: weighted loop
  // 56.4 -> 55.6 ms, identity 46.6 -> 48.3 ms with that order). Claiming the
  // last G tiles as 2-column halves (a shorter last wave, same bits) measured
  // slower: 46.3 -> 47.8 ms.
  auto x_tile = [&](long long tx, long long& g, long long& s) {
    if (DIAG) {
      const long long nf = (nx / S) * (S - 1);   // tiles of chunks 0..S-2
      g = (tx < nf) ? tx / (S - 1) : tx - nf;
      s = (tx < nf) ? tx - g * (S - 1) : S - 1;
    } else {
      // tx / S by a double reciprocal and a +-1 fix (exact for tx < 2^52);
      // an integer division is a long emulated sequence per tile
      g = (long long)((double)tx * rS);
      if (g * S > tx) --g;
      else if ((g + 1) * S <= tx) ++g;
      s = tx - g * S;
    }
  };
  unsigned dummy_nf = 0, dummy_nz = 0;
  // Phase timing and the step trace (tools/ab_arms.py --phases,
  // tools/trace_report.py) are compiled in only with -DRBD_INSTRUMENT=1: their
  // per-call checks were ~3% of the loop's issued instructions (ncu source
  // counters, C2), on the X-tile path.
  constexpr bool kInstr = RBD_INSTRUMENT;
  const bool timing = kInstr && (a.phase_ns != nullptr) && cta == 0 && tid == 0;
  unsigned long long tp = timing ? globaltimer() : 0ull;
  auto mark = [&](int slot) {
    if (kInstr && timing) {
      const unsigned long long t = globaltimer();
      a.phase_ns[slot] += t - tp;
      tp = t;
    }
  };
  unsigned long long* trow = (kInstr && a.trace) ? a.trace + (size_t)cta * kTraceWords : nullptr;
  // tag: 1 P1 start, 2 P1 end, 3 bar1 out, 4 tile start (|tile<<8), 5 tile end,
  //      6 P2 end, 7 bar2 out, 8 P3 end, 9 bar3 out, 10 step end
  auto trace = [&](long long step, unsigned long long tag) {
    if (kInstr && trow && tid == 0 && step >= a.trace_step && step < a.trace_step + 2) {
      const unsigned long long c = trow[0];
      if (c + 1 < kTraceWords) {
        trow[1 + c] = (tag << 40) | (globaltimer() & 0xFFFFFFFFFFull);
        trow[0] = c + 1;
      }
    }
  };

  // the shares start at zero here and are rezeroed as P1 publishes them
  // (zeroing them at the top of each step made ptxas interleave the X-tile
  // batch, as above)
  if (FC && a.fold_kmax > 0)
    for (long long l = tid; l < kNHalf * a.d_max; l += kThreads) psh()[l] = 0.0;   // read after P1's barriers
  while (true) {
    const int live = !done;
    if (!live && !pending) break;
    // =================== P1: w1 = x - Y c (and column k-1's second pass) ===========
    const long long kb = pending ? k - 1 : k;
    trace(k, 1);
    const long long kpad = (k + kPBatch - 1) / kPBatch * kPBatch;
    for (long long l = tid; l < kpad; l += kThreads) {
      cs[l] = (!live || l >= k) ? 0.0
              : SHARD           ? __ldcg(&pay[kPayHead + m + l])
                                : __ldcg(&a.T[l * n + jstar]);
      ps[l] = (pending && reorth_prev && l < kb) ? __ldcg(&pbuf(k - 1)[l]) : 0.0;
    }
    // FOLD: this step forms p_k in P1 (its Y'w1 groups sum the CTA shares)
    const bool fold = FC && live && k > 0 && k <= a.fold_kmax;
    const double* x = SHARD ? pay + kPayHead : a.X + jstar * a.ldx;
    const float* xf = XF32 ? a.Xf + jstar * a.ldx : nullptr;
    __syncthreads();
    double nacc = 0.0, nacc2 = 0.0;
    for (long long rb = r_lo; rb < r_hi; rb += kPRows) {
      // lane owns rows i0 .. i0+VEC-1 of its half (a 16-byte pair when VEC == 2)
      const int half = warp / kPW, wh = warp % kPW;
      const long long i0 = rb + (long long)half * kPHalf + (long long)VEC * lane;
      const long long iend = (rb + kPRows < r_hi) ? rb + kPRows : r_hi;   // rows of this block
      // the first warp of each half finishes the half's rows: their x and
      // w1_{k-1} loads go out now and land while the block's Y batches stream
      double xpre[VEC], wpre[VEC], apre[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const bool in = wh == 0 && i0 + v < iend;
        if constexpr (XF32)
          xpre[v] = (in && live) ? (double)__ldcg(&xf[i0 + v]) : 0.0;
        else
          xpre[v] = (in && live) ? __ldcg(&x[i0 + v]) : 0.0;
        wpre[v] = (in && pending) ? __ldcg(&a.w[i0 + v]) : 0.0;
        if constexpr (DIAG) apre[v] = (in && live) ? __ldg(&a.diag[i0 + v]) : 0.0;
      }
      double acc_c[VEC], acc_p[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc_c[v] = acc_p[v] = 0.0;
      // rows this lane owns in the block (VEC, fewer at an odd tail, or none);
      // every lane keeps 16 predicated loads in flight per batch, including the
      // last partial batch (a serial remainder costs one L2 round trip per column)
      const long long nv_ = iend - i0;
      const int nv = nv_ >= VEC ? VEC : (nv_ > 0 ? (int)nv_ : 0);
      if (nv > 0) {
        const double* yp = a.Y + i0 + (long long)wh * m;
        const long long stp = (long long)kPW * m;
        for (long long l = wh; l < kb; l += kPLoads * kPW) {
          double yv[kPLoads][VEC];
#pragma unroll
          for (int q = 0; q < kPLoads; ++q) {
            const bool ok = l + q * kPW < kb;
            if constexpr (VEC == 2) {
              if (ok && nv == 2) {
                const double2 t2 = __ldcg(reinterpret_cast<const double2*>(yp + q * stp));
                yv[q][0] = t2.x;
                yv[q][VEC - 1] = t2.y;
              } else {
                yv[q][0] = ok ? __ldcg(yp + q * stp) : 0.0;
                yv[q][VEC - 1] = 0.0;
              }
            } else {
              yv[q][0] = ok ? __ldcg(yp + q * stp) : 0.0;
            }
          }
#pragma unroll
          for (int q = 0; q < kPLoads; ++q)
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
              acc_c[v] = fma(yv[q][v], cs[l + q * kPW], acc_c[v]);   // zero past kb
              acc_p[v] = fma(yv[q][v], ps[l + q * kPW], acc_p[v]);
            }
          yp += kPLoads * stp;
        }
      }
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        red_c[warp][VEC * lane + v] = acc_c[v];
        red_p[warp][VEC * lane + v] = acc_p[v];
      }
      __syncthreads();
      if (wh == 0) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const long long i = i0 + v;
          if constexpr (FC) w1s[half * kPHalf + VEC * lane + v] = 0.0;
          if (i >= iend) break;
          const int w0 = half * kPW;
          double sc = red_c[w0][VEC * lane + v], sp = red_p[w0][VEC * lane + v];
#pragma unroll
          for (int w = 1; w < kPW; ++w) {
            sc += red_c[w0 + w][VEC * lane + v];
            sp += red_p[w0 + w][VEC * lane + v];
          }
          if (pending) {
            const double yk1 = (wpre[v] - sp) / wnorm_prev;  // second pass of column k-1
            a.Y[i + (k - 1) * m] = yk1;
            sc = fma(yk1, cs[k - 1], sc);
          }
          if (live) {
            const double w1 = xpre[v] - sc;                  // first pass of column k
            a.w[i] = w1;
            if constexpr (FC) w1s[half * kPHalf + VEC * lane + v] = w1;
            nacc = fma(w1, w1, nacc);
            if constexpr (DIAG) {
              const double awv = apre[v] * w1;               // a o w1 (weight.cpp:83)
              a.aw[i] = awv;
              nacc2 = fma(awv, w1, nacc2);
            }
          }
        }
      }
      __syncthreads();
      if constexpr (FC) {
        // the block's share of p_k = Y[:, 0:k]' w1_k: re-read the block (L2;
        // column k-1 was just written above), a lane's two rows times w1, and a
        // transposing butterfly leaves lane pair 2c..2c+1 with column c of the
        // 16-column batch summed over the half's 64 rows. The most recently
        // read batches are re-read first once k is large (fewer L2 misses).
        if (fold)
          fold_block_share<kPW>(a.Y + i0, m, k, wh, lane, w1s[half * kPHalf + VEC * lane],
                                w1s[half * kPHalf + VEC * lane + 1], nv == 2, psh() + half * a.d_max);
        __syncthreads();
      }
    }
    pending = 0;
    if (!live) continue;   // materialisation-only pass after the stop
    if constexpr (FC) {
      if (fold)   // published by the release-adds below
        for (long long l = tid; l < k; l += kThreads) {
          // read and rezero (the shares start at zero: kernel entry, then here)
          double v = psh()[l];
          psh()[l] = 0.0;
#pragma unroll
          for (int h = 1; h < kNHalf; ++h) {
            v += psh()[h * a.d_max + l];
            psh()[h * a.d_max + l] = 0.0;
          }
          a.ppart[(long long)cta * a.d_max + l] = v;
        }
    }
    {
      const double sblk = block_sum_fixed<kThreads>(warp % kPW == 0 ? nacc : 0.0, smn);
      if constexpr (DIAG) {
        const double sblk2 = block_sum_fixed<kThreads>(warp % kPW == 0 ? nacc2 : 0.0, smn);
        if (tid == 0) a.npart2[cta] = sblk2;
      }
      // block_sum_fixed ends with __syncthreads: every P1 write of this CTA
      // (w1 rows, Y column k-1 rows) precedes the release-adds below
      if (tid == 0) {
        a.npart[cta] = sblk;
        if (r_lo < r_hi)
          for (long long sc = r_lo / kChunk; sc * kChunk < r_hi; ++sc) {
            const long long lo = sc * kChunk > r_lo ? sc * kChunk : r_lo;
            const long long hi = (sc + 1) * kChunk < r_hi ? (sc + 1) * kChunk : r_hi;
            red_release_add_u64(&a.rdy[1 + sc], (unsigned long long)(hi - lo));
          }
        red_release_add_u64(&a.rdy[0], 1ull);
      }
    }
    const unsigned long long ord = (unsigned long long)(k - k_base + 1);   // P1s published so far
    bool all_rdy = false;   // (tid 0) every CTA is through this step's P1
    auto wait_ge = [&](const unsigned long long* c, unsigned long long want) {
      if (ld_acquire_u64(c) >= want) return;
      const unsigned long long t0 = globaltimer();
      unsigned spins = 0;
      do {
        __nanosleep(32);
        if ((++spins & 0xfffu) == 0 && globaltimer() - t0 > 30000000000ull) __trap();
      } while (ld_acquire_u64(c) < want);
    };
    // claim index t -> Y'w1 group (t_y >= 0) or X tile index (t_x >= 0), for a
    // step with gyv Y'w1 groups and totv claims in all
    auto split = [&](long long t, long long gyv, long long totv, long long& t_y, long long& t_x) {
      const long long nxv = totv - gyv;
      const long long yo = DIAG ? 0 : (a.ydelay < nxv ? a.ydelay : nxv);
      if (t < yo) {
        t_y = -1;
        t_x = t;
      } else if (t < yo + gyv) {
        t_y = t - yo;
        t_x = -1;
      } else {
        t_y = -1;
        t_x = t - gyv;
      }
    };
    // (tid 0, before publishing tile t to the CTA) the P1 rows tile t reads
    auto wait_inputs = [&](long long t, long long gy_, long long total_) {
      if (t >= total_ || all_rdy) return;
      if (ld_acquire_u64(&a.rdy[0]) >= (unsigned long long)G * ord) {
        all_rdy = true;
        return;
      }
      long long t_y, t_x;
      split(t, gy_, total_, t_y, t_x);
      if (t_y >= 0) {
        wait_ge(&a.rdy[0], (unsigned long long)G * ord);
        all_rdy = true;
      } else {
        long long gx, sc;
        x_tile(t_x, gx, sc);
        const long long rows = (m - sc * kChunk < kChunk) ? m - sc * kChunk : kChunk;
        wait_ge(&a.rdy[1 + sc], (unsigned long long)rows * ord);
      }
    };
    mark(0);
    trace(k, 2);
    trace(k, 3);
    mark(1);

    // =================== P2: one dynamic queue of tiles ===================
    //   [0, gy)       Y' w1 column groups, full height -> p_k[4g..4g+3] (the
    //                 reorth coefficients) summed over chunks in order by one
    //                 CTA; the last one to finish decides the second pass
    //                 (decompose.cpp:28), ||w_k|| and breakdown (:29-30)
    //   [gy, gy+nx)   X' w1 tiles (the fused sweep), group-major (DIAG: chunks
    //                 0..S-2 group-major, then every group's last chunk). The
    //                 claimer of a group's last chunk finalises the group in-queue:
    //                 T[k, j] = (w1.x_j - p.T[0:k, j]) / ||w_k||, residuals
    //                 (workspace.cpp:52-53). Chunk partials double as ready
    //                 flags (NaN = not written); the siblings were claimed
    //                 earlier and finalisation is deferred by one tile, so the
    //                 poll rarely waits, and every wait targets an
    //                 earlier-claimed tile (no deadlock).
    const long long gy = (FC && k > 0 && k <= a.fold_kmax) ? (k + kFoldCols - 1) / kFoldCols
                                                            : (k + kCols - 1) / kCols;
    const long long total = gy + nx;
    double bv = -1.0;          // this CTA's best finalised residual (argmax record)
    long long bj = 0x7fffffffffffffffLL;
    if (gy == 0 && cta == 0 && tid == 0) {   // k == 0: nothing to orthogonalise against
      wait_ge(&a.rdy[0], (unsigned long long)G * ord);
      double w1n2 = 0.0;
      for (int b = 0; b < G; ++b) w1n2 += __ldcg(&a.npart[b]);
      const double norm0 = sqrt(w1n2);
      ctl->norm = norm0;
      ctl->reorth = 0;
      ctl->breakdown = (norm0 < tol || norm0 == 0.0) ? 1 : 0;
      if constexpr (DIAG) {   // YAY[0, 0] = w1'Aw1 / ||w1||^2
        double w1a = 0.0;
        for (int b = 0; b < G; ++b) w1a += __ldcg(&a.npart2[b]);
        const double y00 = w1a / (norm0 * norm0);
        a.yrow[0] = y00;
        a.YAY[0] = y00;
        __threadfence();
      }
      st_release_s64(&ctl->p_step, k + 1);
      if (DIAG) st_release_s64(&ctl->y_step, k + 1);
    }
    // Groups whose last chunk this CTA swept and that are not finalised yet
    // (FIFO, uniform across the CTA). Finalisation is attempted after the next
    // tile without waiting; it blocks only when the FIFO is full or the queue
    // is exhausted. Every wait targets an earlier-claimed tile (a sibling
    // chunk, or the Y'w1 groups that precede all X tiles): no cycles.
    // pending-group FIFO depth and when a tile's finalisation attempt runs
    // (before or after the tile's own group is queued): measured per loop,
    // C1 fp64 46.3 -> 46.1 ms and weighted 55.8 -> 55.3 ms with (2, after);
    // the fp32 loop keeps (4, before): 33.8 ms against 34.6 ms
#ifndef RBD_F32_PEND
#define RBD_F32_PEND 4
#endif
#ifndef RBD_F32_FINFIRST
#define RBD_F32_FINFIRST 1
#endif
    constexpr int kPend = XF32 ? RBD_F32_PEND : 2;
    constexpr bool kFinFirst = XF32 && RBD_F32_FINFIRST;
    long long pend[kPend];
#pragma unroll
    for (int i = 0; i < kPend; ++i) pend[i] = -1;
    int npend = 0;
    // the step's published decision, read once per CTA
    bool p_ready = false;
    int re_s = 0, bd_s = 0;
    double nrm_s = 1.0;
    auto ensure_p = [&](const bool block) -> bool {
      if (p_ready) return true;
      if (tid == 0) {
        int ok = ld_acquire_s64(&ctl->p_step) == k + 1;
        if (!ok && block) {
          wait_step(&ctl->p_step, k + 1);
          ok = 1;
        }
        sh_ok = ok;
      }
      __syncthreads();
      if (!sh_ok) return false;
      re_s = __ldcg(&ctl->reorth);
      bd_s = __ldcg(&ctl->breakdown);
      nrm_s = __ldcg(&ctl->norm);
      if constexpr (DIAG) {
        if (!bd_s) {
          for (long long l = tid; l <= k; l += kThreads)
            pd[l] = (re_s && l < k) ? __ldcg(&pbuf(k)[l]) : 0.0;
          __syncthreads();
        }
      }
      p_ready = true;
      return true;
    };
    // DIAG: the YAY row YAY[k, 0:k+1] (see the header), distributed: slice sl
    // (kYSlice entries, one warp per entry l) is computed by CTA sl % G once
    // the decision is out: v_l = YAY[l, 0:k] . p (lane-strided, xor-butterfly),
    // YAY[k, l] = (q_l - v_l) / ||w|| (q_l when there is no second pass); the
    // slice's p.q and p.v go to yslice[sl]. The CTA completing the last slice
    // sums them in slice order for YAY[k, k] and publishes the row. Every CTA
    // does its slices before it waits on the row or on the step barrier, so
    // no wait can cycle.
    bool y_mine = false, y_ready = false;
    auto yay_slices = [&](const bool block) {
      if (!DIAG || y_mine) return;
      if (k == 0) {   // row [YAY[0, 0]] published with the decision
        y_mine = true;
        return;
      }
      if (!ensure_p(block)) return;
      y_mine = true;
      if (bd_s) return;
      const long long ld = a.d_max;
      const long long nsl = (k + kYSlice - 1) / kYSlice;
      for (long long sl = cta; sl < nsl; sl += G) {
        const long long l = sl * kYSlice + warp;
        double v = 0.0;
        if (re_s && l < k)
          for (long long mm = lane; mm < k; mm += 32) v = fma(__ldcg(&a.YAY[l * ld + mm]), pd[mm], v);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) smn[warp] = v;
        __syncthreads();
        if (tid == 0) {
          double pq = 0.0, pv = 0.0;
          for (int w = 0; w < kYSlice; ++w) {
            const long long ll = sl * kYSlice + w;
            if (ll >= k) break;
            const double ql = __ldcg(a.q + ll), vl = smn[w];
            const double yl = (re_s ? ql - vl : ql) / nrm_s;
            a.yrow[ll] = yl;
            a.YAY[k * ld + ll] = yl;
            a.YAY[ll * ld + k] = yl;
            if (re_s) {
              pq = fma(pd[ll], ql, pq);
              pv = fma(pd[ll], vl, pv);
            }
          }
          a.yslice[2 * sl] = pq;
          a.yslice[2 * sl + 1] = pv;
        }
        __syncthreads();
      }
      if (tid == 0) {
        __threadfence();
        if (atomicAdd(&ctl->yslices, 1u) == (unsigned)(G - 1)) {   // last: YAY[k, k]
          __threadfence();
          double pq = 0.0, pv = 0.0;
          for (long long sl = 0; sl < nsl; ++sl) {
            pq += __ldcg(&a.yslice[2 * sl]);
            pv += __ldcg(&a.yslice[2 * sl + 1]);
          }
          const double w1a = __ldcg(&ctl->w1a);
          const double num = re_s ? (w1a - 2.0 * pq) + pv : w1a;
          const double ykk = num / (nrm_s * nrm_s);
          a.yrow[k] = ykk;
          a.YAY[k * ld + k] = ykk;
          ctl->yslices = 0u;
          __threadfence();
          st_release_s64(&ctl->y_step, k + 1);
        }
      }
      trace(k, 12);
    };
    auto ensure_y = [&](const bool block) -> bool {
      if (y_ready) return true;
      yay_slices(block);
      if (!y_mine) return false;
      if (bd_s) {
        y_ready = true;
        return true;
      }
      if (tid == 0) {
        int ok = ld_acquire_s64(&ctl->y_step) == k + 1;
        if (!ok && block) {
          wait_step(&ctl->y_step, k + 1);
          ok = 1;
        }
        sh_ok = ok;
      }
      __syncthreads();
      if (!sh_ok) return false;
      for (long long l = tid; l <= k; l += kThreads) yd[l] = __ldcg(&a.yrow[l]);
      __syncthreads();
      y_ready = true;
      return true;
    };
    // Finalise up to two groups at once (warps 0-3: pend[0], warps 4-7:
    // pend[1]; one column per warp): all loads of the pass are issued together.
    // Groups whose chunk partials are not all written yet (a NaN sum) are kept
    // unless block. Returns the number of groups retired from the FIFO front.
    auto finalize_pass = [&](const bool block) {
      if (!ensure_p(block)) return;
      if (DIAG && !ensure_y(block)) return;
      const int q = warp >> 2;
      const long long g = q < npend ? pend[q] : -1;
      const long long j = g * kCols + (warp & 3);
      const bool mine = g >= 0 && j < n;
      double sp = 0.0, corr = 0.0, rj = 0.0;
      double sp2 = 0.0, corr2 = 0.0, gg = 0.0;   // DIAG: (a o w1).x_j, p.YAX[:, j], YAY row . T[:, j]
      double cr0 = 0.0, qd0 = 0.0, ca0 = 0.0;      // DIAG (lane 0): cross_j, quad_j, col_sq_A[j]
      if (mine) {   // a chunk partial not written yet is NaN, and so is the sum
        for (long long ss = lane; ss < S; ss += 32) sp += ld_relaxed_f64(&a.partial[ss * n + j]);
        if constexpr (DIAG) {
          // every load of the pass goes out before any is used: one L2 round trip
          for (long long ss = lane; ss < S; ss += 32) sp2 += ld_relaxed_f64(&a.partial2[ss * n + j]);
          if (lane == 0) {   // carried sums: only this group's finaliser writes them
            cr0 = __ldcg(&a.cross[j]);
            qd0 = __ldcg(&a.quad[j]);
            ca0 = __ldg(&a.colsq_a[j]);
          }
          if (!bd_s) {
            for (long long l0 = 0; l0 < k; l0 += 256) {
              double tv[8], av[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const long long l = l0 + lane + 32 * u;
                tv[u] = (l < k) ? __ldcg(&a.T[l * n + j]) : 0.0;
                av[u] = (l < k && re_s) ? __ldcg(&a.YAX[l * n + j]) : 0.0;
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const long long l = l0 + lane + 32 * u;
                const double pl = (l < k) ? pd[l] : 0.0, yl = (l < k) ? yd[l] : 0.0;
                corr = fma(pl, tv[u], corr);
                corr2 = fma(pl, av[u], corr2);
                gg = fma(yl, tv[u], gg);
              }
            }
          }
          sp = (sp2 == sp2) ? sp : sp2;   // NaN if either row is incomplete
        } else if (lane == 0) {
          rj = __ldcg(&a.r[j]);
        }
        if (!DIAG && re_s && !bd_s) {
          for (long long l0 = 0; l0 < k; l0 += 512) {
            double tv[16], pv[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              const long long l = l0 + lane + 32 * u;
              tv[u] = (l < k) ? __ldcg(&a.T[l * n + j]) : 0.0;
              pv[u] = (l < k) ? __ldcg(&pbuf(k)[l]) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) corr = fma(pv[u], tv[u], corr);
          }
        }
      }
      const bool nr0 = __syncthreads_or(mine && q == 0 && sp != sp);
      const bool nr1 = __syncthreads_or(mine && q == 1 && sp != sp);
      bool commit = mine && !(q == 0 ? nr0 : nr1);
      if (block && mine && !commit) {
        sp = 0.0;
        for (long long ss = lane; ss < S; ss += 32) sp += poll_f64(&a.partial[ss * n + j]);
        if constexpr (DIAG) {
          sp2 = 0.0;
          for (long long ss = lane; ss < S; ss += 32) sp2 += poll_f64(&a.partial2[ss * n + j]);
        }
        commit = true;
      }
      if (commit) {
        for (long long ss = lane; ss < S; ss += 32) st_relaxed_f64(&a.partial[ss * n + j], kNaN);
        if constexpr (DIAG)
          for (long long ss = lane; ss < S; ss += 32) st_relaxed_f64(&a.partial2[ss * n + j], kNaN);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          sp += __shfl_xor_sync(0xffffffffu, sp, off);
          corr += __shfl_xor_sync(0xffffffffu, corr, off);
          if constexpr (DIAG) {
            sp2 += __shfl_xor_sync(0xffffffffu, sp2, off);
            corr2 += __shfl_xor_sync(0xffffffffu, corr2, off);
            gg += __shfl_xor_sync(0xffffffffu, gg, off);
          }
        }
        if (DIAG && lane == 0 && !bd_s) {
          // weighted bookkeeping (rbd_weighted.cuh; workspace.cpp:61-99)
          const double tt = (sp - corr) / nrm_s;                 // decompose.cpp:93
          const double ya = (sp2 - corr2) / nrm_s;               // workspace.cpp:66
          a.T[k * n + j] = tt;
          a.YAX[k * n + j] = ya;
          const double cr = cr0 + tt * ya;
          const double qd = qd0 + (2.0 * tt * gg + yd[k] * tt * tt);
          a.cross[j] = cr;
          a.quad[j] = qd;
          double e2 = ca0 - 2.0 * cr + qd;                       // workspace.cpp:88-97
          e2 = e2 > 0.0 ? e2 : 0.0;
          if (rec_better(e2, j, bv, bj)) {
            bv = e2;
            bj = j;
          }
        } else if (!DIAG && lane == 0 && !bd_s) {
          const double tt = (sp - corr) / nrm_s;
          a.T[k * n + j] = tt;                                   // decompose.cpp:93
          const double sq = __dmul_rn(tt, tt);
          double rr = __dsub_rn(rj, sq);                         // workspace.cpp:52-53
          rr = rr > 0.0 ? rr : 0.0;
          a.r[j] = rr;
          if (rec_better(rr, j, bv, bj)) {
            bv = rr;
            bj = j;
          }
        }
      }
      // retire committed groups (uniform: nr0/nr1 are CTA-wide)
      const bool ok0 = npend > 0 && (block || !nr0);
      const bool ok1 = npend > 1 && (block || !nr1);
      int w = 0;
      for (int i = 0; i < npend; ++i)
        if (!((i == 0 && ok0) || (i == 1 && ok1))) pend[w++] = pend[i];
      npend = w;
    };
    long long next = 0;
    if (tid == 0) next = (long long)(atomicAdd(&ctl->tile_ctr, 1ull) - tile_base);
    while (true) {
      mark(9);
      if (tid == 0) {
        wait_inputs(next, gy, total);   // acquire by tid 0, published by the barrier below
        // published as: -1 - g for Y'w1 group g, the X tile index, or total (end)
        long long t_y, t_x;
        split(next, gy, total, t_y, t_x);
        sh_tile = next >= total ? total : (t_y >= 0 ? -1 - t_y : t_x);
      }
      __syncthreads();
      const long long code = sh_tile;
      mark(5);
      if (code >= total) break;
      trace(k, 4 | ((unsigned long long)(code < 0 ? -1 - code : code + gy) << 8));
      if (tid == 0) next = (long long)(atomicAdd(&ctl->tile_ctr, 1ull) - tile_base);
      if (code < 0) {
        const long long t = -1 - code;   // the Y'w1 group
        if (FC && k <= a.fold_kmax)   // a FOLD step (k > 0 here)
          fold_group_sum(a.ppart, a.d_max, G, k, t, &red_c[0][0], pbuf(k));
        else
        for (long long s = 0; s < S; ++s) {
          if constexpr (DIAG)
            sweep_tile_dot2<VEC, LOAD_CG, true, 2>(a.Y, m, m, k, a.w, a.aw, a.ppart, a.ppart2,
                                                   a.d_max, s * gy + t, red2);
          else
            sweep_tiles<VEC, MODE_DOT, LOAD_CG, true>(a.Y, m, m, k, a.w, a.ppart, a.d_max,
                                                       s * gy + t, 1LL << 40, red, dummy_nf,
                                                       dummy_nz);
        }
        // the partials of this group were written by this CTA (CTA-visible)
        if (!(FC && k <= a.fold_kmax) && tid < kCols && t * kCols + tid < k) {
          const long long l = t * kCols + tid;
          double v = 0.0;
          for (long long s = 0; s < S; ++s) v += a.ppart[s * a.d_max + l];
          pbuf(k)[l] = v;
          if constexpr (DIAG) {
            double v2 = 0.0;
            for (long long s = 0; s < S; ++s) v2 += a.ppart2[s * a.d_max + l];
            a.q[l] = v2;
          }
        }
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          sh_tile = (atomicAdd(&ctl->ydone, 1u) == (unsigned)(gy - 1)) ? 1 : 0;
          if (sh_tile) __threadfence();
        }
        __syncthreads();
        if (sh_tile) {
          // decider: ||p||^2, ||w1||^2, the second-pass condition, ||w||, breakdown
          double pn = 0.0;
          for (long long ll = tid; ll < k; ll += kThreads) {
            const double pv = __ldcg(&pbuf(k)[ll]);
            pn = fma(pv, pv, pn);
          }
          pn = block_sum_fixed<kThreads>(pn, smn);
          double w1n2 = 0.0;
          for (int b = tid; b < G; b += kThreads) w1n2 += __ldcg(&a.npart[b]);
          w1n2 = block_sum_fixed<kThreads>(w1n2, smn);
          double w1a = 0.0;
          if constexpr (DIAG) {
            for (int b = tid; b < G; b += kThreads) w1a += __ldcg(&a.npart2[b]);
            w1a = block_sum_fixed<kThreads>(w1a, smn);
          }
          const int re = (cfg_reorth || sqrt(w1n2) < 0.5 * sqrt(xnorm2)) ? 1 : 0;    // :28
          double wn2 = re ? w1n2 - pn : w1n2;
          if (re && wnorm_in_guard_band(wn2, w1n2, pn, tol))   // decide on the exact ||w||
            wn2 = exact_wnorm2<kThreads>(a.w, a.Y, m, m, k, pbuf(k), smn);
          if (tid == 0) {
            ctl->ydone = 0u;
            wn2 = wn2 > 0.0 ? wn2 : 0.0;
            const double nrm = sqrt(wn2);
            const int bd = (nrm < tol || nrm == 0.0) ? 1 : 0;                       // :29-30
            ctl->norm = nrm;
            ctl->reorth = re;
            ctl->breakdown = bd;
            sh_dec[0] = re;
            sh_dec[1] = bd;
            sh_decd[0] = nrm;
            if (DIAG) ctl->w1a = w1a;
            st_release_s64(&ctl->p_step, k + 1);
          }
          trace(k, 11);
        }
        mark(6);
        trace(k, 5);
      } else {
        // X tiles group-major (contiguous column runs per group); the claimer of
        // a group's last chunk finalises it after its NEXT tile (deferred), so
        // the siblings are long done and finalisation never piles up at the
        // end of the queue
        long long g, s;
        x_tile(code, g, s);
        if constexpr (DIAG && VEC == 2)
        {
          sweep_tile_dot2_sv<LOAD_STREAM, kSvUB, false>(a.X, a.ldx, m, n, a.w, a.aw, a.partial,
                                                        a.partial2, n, s, g, red2, svec);
          if (s == S - 1) __syncthreads();   // only before a finalisation of this chunk
        }
        else if constexpr (DIAG)
          sweep_tile_dot2<VEC, LOAD_STREAM, true, 2>(a.X, a.ldx, m, n, a.w, a.aw, a.partial,
                                                     a.partial2, n, s * ngx + g, red2);
        else if constexpr (XF32)   // g: an 8-column tile = finalisation groups 2g, 2g+1
        {
          sweep_tiles_f32<MODE_DOT, true, kXT, false>(a.Xf, a.ldx, m, n, a.w, a.partial, n,
                                                      s * ngt + g, 1LL << 40, red2, dummy_nf,
                                                      dummy_nz, a.xvec4 != 0);
          if (s == S - 1) __syncthreads();   // as below: only before a finalisation of this chunk
        }
        else
          // the load-batch fence keeps each X batch whole where ptxas split
          // it (sharded, FOLD: FMAs between the loads in SASS); the base
          // kernel issues whole batches without it, and there the fence's
          // later start of the FMAs cost C1 2.5% (batch_fence)
        {
          sweep_tile<VEC, MODE_DOT, LOAD_STREAM, true, kCols, SHARD || FOLD>(a.X, a.ldx, m, n, a.w, a.partial,
                                                                          n, s, g, red, dummy_nf, dummy_nz);
          // the claim barrier orders `red` for the next tile; a barrier here
          // only when the finalisation attempt below may read this tile's own
          // chunk partials (the group's last chunk)
          if (s == S - 1) __syncthreads();
        }
        mark(7);
        if (DIAG) yay_slices(false);   // this CTA's share of the YAY row, once decided
        if (kFinFirst && npend > 0) finalize_pass(false);
        if (s == S - 1) {
          constexpr int per = kXT / kCols;   // finalisation groups this tile completes
          if (npend > kPend - per) finalize_pass(true);   // retire the two oldest
          for (int h = 0; h < per; ++h)
            if (g * per + h < ngx) pend[npend++] = g * per + h;
        }
        if (!kFinFirst && npend > 0) finalize_pass(false);
        trace(k, 5);
      }
    }
    while (npend > 0) finalize_pass(true);
    if (DIAG) yay_slices(true);   // others may be waiting on this CTA's slices
    block_argmax<kThreads>(bv, bj, smr);
    if (tid == 0) a.rec[cta] = Rec{bv, bj};
    tile_base += (unsigned long long)(total + G);
    mark(2);
    trace(k, 6);
    grid_barrier(a.bar, gen);
    trace(k, 7);
    mark(3);
    // columns [0, k) of Y (column k-1 materialised in this step's P1) are
    // written at GPU scope: a copy engine may fetch them while the loop runs
    if (a.progress && cta == 0 && tid == 0) *(volatile long long*)a.progress = k;
    if constexpr (SHARD) {   // every claim of this launch is done: rezero for the next launch
      if (cta == 0 && tid == 0) ctl->tile_ctr = 0ull;
    }

    // every CTA: the published decision, the global argmax over the CTA
    // records (workspace.cpp:107-113,123) and the stop test (decompose.cpp:87)
    {
      // one round trip for all of it: the decision words and the CTA records
      const int bd = __ldcg(&ctl->breakdown);
      const double nrm = __ldcg(&ctl->norm);
      const int re = __ldcg(&ctl->reorth);
      double rv0 = -1.0, rv1 = -1.0;
      long long rj0 = 0x7fffffffffffffffLL, rj1 = 0x7fffffffffffffffLL;
      if (tid < G) {
        rv0 = __ldcg(&a.rec[tid].v);
        rj0 = __ldcg(&a.rec[tid].j);
      }
      if (tid + kThreads < G) {
        rv1 = __ldcg(&a.rec[tid + kThreads].v);
        rj1 = __ldcg(&a.rec[tid + kThreads].j);
      }
      if (bd) {                        // decompose.cpp:90 — keep the d we have
        done = 1;
        breakdown = 1;
        if constexpr (SHARD) {
          if (cta == 0 && tid == 0) {
            st->breakdown = 1;
            st->done = 1;
            st->pending = 0;
          }
          break;
        }
        continue;
      }
      double gv = -1.0;
      long long gj = 0x7fffffffffffffffLL;
      if (rec_better(rv0, rj0, gv, gj)) {
        gv = rv0;
        gj = rj0;
      }
      if (rec_better(rv1, rj1, gv, gj)) {
        gv = rv1;
        gj = rj1;
      }
      for (int b = tid + 2 * kThreads; b < G; b += kThreads) {   // grids above 512 CTAs
        const double v = __ldcg(&a.rec[b].v);
        const long long jj = __ldcg(&a.rec[b].j);
        if (rec_better(v, jj, gv, gj)) {
          gv = v;
          gj = jj;
        }
      }
      block_argmax<kThreads>(gv, gj, smr);
      if constexpr (SHARD) {
        // this rank's 16-byte record {best residual, global index}; after the
        // record allgather the owner of the winner packs x_j and T[0:k+1, j]
        // (k_shard_pack) for the payload allreduce
        const bool have = gj != 0x7fffffffffffffffLL;
        if (cta == 0 && tid == 0) {
          a.send[0] = have ? gv : -2.0;
          a.send[1] = __longlong_as_double(have ? a.col_offset + gj : -1LL);
          st->jlocal = have ? gj : -1;
          st->reorth = re;
          st->wnorm = nrm;
          st->pending = 0;
        }
        break;
      } else {
        e_cur = sqrt(gv > 0.0 ? gv : 0.0);
        if (cta == 0 && tid == 0) {
          a.selected[k] = jstar;         // decompose.cpp:94
          a.history[k] = e_cur;          // :99
        }
        k += 1;                          // :96
        pending = 1;
        reorth_prev = re;
        wnorm_prev = nrm;
        jstar = (k < a.nforced) ? __ldg(&a.forced[k]) : gj;   // :101 (forced: parity re-run)
        xnorm2 = a.col_sq[jstar];        // entry norm of the column extended next (:18)
        done =!(k < a.d_max && e_cur > eps_R) ? 1 : 0;   // :87
      }
    }
    trace(k - 1, 10);
    mark(4);
  }
  if constexpr (SHARD) {
    if (cta == 0 && tid == 0 && !live_at_exit(done, breakdown)) st->pending = 0;
  } else {
    if (cta == 0 && tid == 0) {
      st->d = k;
      st->done = 1;
      st->breakdown = breakdown;
      st->e_cur = e_cur;
      st->jstar = jstar;
    }
  }
}

// Sharded mode, after the record allgather: every rank applies the winner
// rule to the same records (rbd_select.h); the owner packs the winner's
// payload {col_sq, x_j, T[0:k+1, j]} and every other rank contributes -0.0
// (x + -0.0 == x for every x, signed zeros included, so the sum allreduce that
// follows moves the owner's bits exactly, in any order and at any rank count).
static __global__ void k_shard_pack(const DevState* st, const double* rrec, int nranks, int rank,
                                    const double* X, long long ldx, long long m, const double* T,
                                    long long n_local, const double* col_sq, double* pay,
                                    long long pay_count) {
  double bv;
  long long bj;
  const int br = rbdsel::pick(rrec, nranks, 2, &bv, &bj);
  const bool own = !st->done && br == rank;
  const long long jl = own ? st->jlocal : -1;
  const long long k = st->d;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < pay_count; t += stride) {
    double v = -0.0;
    if (own) {
      if (t == 2) v = col_sq[jl];
      else if (t >= kPayHead && t < kPayHead + m) v = X[jl * ldx + (t - kPayHead)];
      else if (t >= kPayHead + m && t <= kPayHead + m + k) v = T[(t - kPayHead - m) * n_local + jl];
    }
    pay[t] = v;
  }
}

// Sharded mode, after the payload allreduce: the step's bookkeeping
// (decompose.cpp:94-101), identical on every rank.
static __global__ void k_shard_select(DevState* st, const double* rrec, const double* pay,
                                      int nranks, double* history, long long* selected) {
  if (threadIdx.x != 0 || st->done) return;
  double bv;
  long long bj;
  rbdsel::pick(rrec, nranks, 2, &bv, &bj);
  const long long k = st->d;
  const double e_cur = sqrt(bv > 0.0 ? bv : 0.0);      // workspace.cpp:123
  history[k] = e_cur;                                   // decompose.cpp:99
  selected[k] = st->jstar;                              // :94
  st->e_cur = e_cur;
  st->d = k + 1;                                        // :96
  st->pending = 1;
  st->jstar = bj;                                       // :101
  st->rank_owner = 0;
  st->xnorm2 = pay[2];
  st->done = !((k + 1) < st->d_max && e_cur > st->eps_R) ? 1 : 0;  // :87
}

// Sharded mode, before step 0: the owner of the start column publishes it
// ({col_sq, x_j0} through the same -0.0-padded allreduce).
static __global__ void k_shard_seed_pack(const double* X, long long ldx, long long m, long long jlocal,
                                         const double* col_sq, double* pay, long long pay_count) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < pay_count; t += stride) {
    double v = -0.0;
    if (jlocal >= 0) {
      if (t == 2) v = col_sq[jlocal];
      else if (t >= kPayHead && t < kPayHead + m) v = X[jlocal * ldx + (t - kPayHead)];
    }
    pay[t] = v;
  }
}

static __global__ void k_shard_seed_select(DevState* st, const double* pay) {
  if (threadIdx.x != 0) return;
  st->rank_owner = 0;
  st->xnorm2 = pay[2];
}

// Virtual ranks (one device): the sum allreduce of the R payloads, in rank
// order, into every rank's receive buffer.
struct PayPtrs {
  const double* in[16];
  double* out[16];
};
static __global__ void k_sum_payloads(PayPtrs p, int nranks, long long count) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) {
    double v = p.in[0][t];
    for (int r = 1; r < nranks; ++r) v += p.in[r][t];
    for (int r = 0; r < nranks; ++r) p.out[r][t] = v;
  }
}

}  // namespace rbdk
