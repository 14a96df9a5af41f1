// rbd_capi.cu — host runtime of the B200 RBD path behind the C ABI in
// include/rbd_cuda.h: context, scratch management, the CUDA-graph-captured
// greedy step loop, the workspace API and out-of-sample projection.
#include "rbd_capi_internal.h"
#include "rbd_persistent.cuh"
#include "rbd_project.cuh"

namespace {
thread_local std::string g_err;
}  // namespace

namespace rbdc {

// ---------------------------------------------------------------------------
// Launch helpers (each increments the context's launch counter)
// ---------------------------------------------------------------------------
int sweep_grid(rbd_ctx_t ctx, long long m, long long ncols_max, int vec) {
  const long long tiles = cdiv(m, kChunk) * cdiv(std::max<long long>(ncols_max, 1), kCols);
  const long long cap = (long long)ctx->nsm * (vec == 2 ? ctx->occ_sweep2 : ctx->occ_sweep1);
  return (int)std::max<long long>(1, std::min(tiles, cap));
}

int launch_sweep(rbd_ctx_t ctx, const SweepArgs& a, int vec, int mode, bool stream_a,
                 long long ncols_max) {
  const int grid = sweep_grid(ctx, a.m, ncols_max, vec);
  if (vec == 2) {
    if (mode == MODE_INIT)
      k_sweep<2, MODE_INIT, true><<<grid, kThreads, 0, ctx->stream>>>(a);
    else if (stream_a)
      k_sweep<2, MODE_DOT, true><<<grid, kThreads, 0, ctx->stream>>>(a);
    else
      k_sweep<2, MODE_DOT, false><<<grid, kThreads, 0, ctx->stream>>>(a);
  } else {
    if (mode == MODE_INIT)
      k_sweep<1, MODE_INIT, true><<<grid, kThreads, 0, ctx->stream>>>(a);
    else if (stream_a)
      k_sweep<1, MODE_DOT, true><<<grid, kThreads, 0, ctx->stream>>>(a);
    else
      k_sweep<1, MODE_DOT, false><<<grid, kThreads, 0, ctx->stream>>>(a);
  }
  ctx->launches++;
  CU(cudaGetLastError());
  return RBD_OK;
}

int finalize_grid(rbd_ctx_t ctx, long long n) {
  return (int)std::max<long long>(1, std::min<long long>(cdiv(n, kThreads), (long long)ctx->nsm * 4));
}

long long gemv_grid(long long m) { return cdiv(m, kGemvRows); }

// ---------------------------------------------------------------------------
// K1: init pass over X (col_sq, residual, flags, max col_sq)
// ---------------------------------------------------------------------------
int enqueue_init_f32(rbd_ctx_t ctx, const float* X, long long m, long long n, long long ldx,
                     double* partial, double* colsq, double* resid, DevState* st) {
  const int vec4 = (ldx % 4 == 0 && aligned16(X)) ? 1 : 0;
  const int grid = sweep_grid(ctx, m, n, 2);
  k_sweep_init_f32<<<grid, kThreads, 0, ctx->stream>>>(X, ldx, m, n, partial, st, vec4);
  ctx->launches++;
  CU(cudaGetLastError());
  const int g = (int)std::max<long long>(1, std::min<long long>(cdiv(n, 256), 1024));
  k_init_finish<<<g, 256, 0, ctx->stream>>>(partial, cdiv(m, kChunk), n, colsq, resid, st);
  ctx->launches++;
  CU(cudaGetLastError());
  return RBD_OK;
}

int enqueue_init(rbd_ctx_t ctx, const double* X, long long m, long long n, long long ldx,
                 double* partial, double* colsq, double* resid, DevState* st) {
  const int vec = (ldx % 2 == 0 && aligned16(X)) ? 2 : 1;
  SweepArgs a{};
  a.A = X;
  a.lda = ldx;
  a.m = m;
  a.ncols = n;
  a.partial = partial;
  a.pstride = n;
  a.st = st;
  a.gate = GATE_NONE;
  TRY(launch_sweep(ctx, a, vec, MODE_INIT, true, n));
  const int g = (int)std::max<long long>(1, std::min<long long>(cdiv(n, 256), 1024));
  k_init_finish<<<g, 256, 0, ctx->stream>>>(partial, cdiv(m, kChunk), n, colsq, resid, st);
  ctx->launches++;
  CU(cudaGetLastError());
  return RBD_OK;
}

// ---------------------------------------------------------------------------
// One extension (K4) on device state: x from X[:, st->jlocal] (or v), first
// coefficients c, basis B = Y[:, 0:st->d] (ld m); result y written to
// ybase + (use_d ? st->d*m : 0).
// ---------------------------------------------------------------------------
struct ExtBufs {
  const double* B;
  long long m;
  long long dcap;       // max basis size (grid sizing of the reorth sweep)
  const double* X;
  long long ldx;
  const double* v;
  const double* c;
  double* w;
  double* p;
  double* nrm;
  double* partial;      // >= S * dcap doubles
  double* ybase;
  int use_d;
  long long* selected;
  DevState* st;
};

int enqueue_extension(rbd_ctx_t ctx, const ExtBufs& b) {
  const long long gb = gemv_grid(b.m);
  ExtArgs e{};
  e.B = b.B;
  e.ldb = b.m;
  e.m = b.m;
  e.X = b.X;
  e.ldx = b.ldx;
  e.v = b.v;
  e.c = b.c;
  e.w = b.w;
  e.nrm_part = b.nrm;
  e.st = b.st;
  e.gate = GATE_LIVE;
  e.pass = 1;
  k_ext_gemv_n<<<(unsigned)gb, kThreads, 0, ctx->stream>>>(e);
  ctx->launches++;
  k_ext_decide<<<1, kThreads, 0, ctx->stream>>>(b.nrm, gb, b.st);
  ctx->launches++;
  // reorth pass: p = B' w (chunked dots over the basis columns), w -= B p
  const int vec = (b.m % 2 == 0 && aligned16(b.B) && aligned16(b.w)) ? 2 : 1;
  SweepArgs s{};
  s.A = b.B;
  s.lda = b.m;
  s.m = b.m;
  s.ncols = b.dcap;
  s.v = b.w;
  s.partial = b.partial;
  s.pstride = b.dcap;
  s.st = b.st;
  s.gate = GATE_REORTH;
  s.csel = 1;
  TRY(launch_sweep(ctx, s, vec, MODE_DOT, false, b.dcap));
  k_coef_combine<<<(unsigned)std::max<long long>(1, cdiv(b.dcap, 256)), 256, 0, ctx->stream>>>(
      b.partial, cdiv(b.m, kChunk), b.dcap, b.p, b.st, GATE_REORTH);
  ctx->launches++;
  e.c = b.p;
  e.gate = GATE_REORTH;
  e.pass = 2;
  k_ext_gemv_n<<<(unsigned)gb, kThreads, 0, ctx->stream>>>(e);
  ctx->launches++;
  k_ext_finish<<<1, kThreads, 0, ctx->stream>>>(b.nrm, gb, b.st, b.selected);
  ctx->launches++;
  const int ng = (int)std::max<long long>(1, std::min<long long>(cdiv(b.m, 256), (long long)ctx->nsm * 8));
  k_normalize<<<ng, 256, 0, ctx->stream>>>(b.w, b.ybase, b.m, b.m, b.st, b.use_d);
  ctx->launches++;
  CU(cudaGetLastError());
  return RBD_OK;
}

struct LoopBufs {
  const double* X;
  long long m, n, ldx, d_max;
  double* Y;
  double* T;
  const float* Xf = nullptr;   // fp32 storage mode (X == nullptr): persistent loop only
};

// One greedy step: extension (K4) + fused sweep (K2) + finalize/argmax (K3).
int diag_vec_grid(rbd_ctx_t ctx, long long m) {
  return (int)std::max<long long>(1, std::min<long long>(cdiv(m, kThreads), (long long)ctx->nsm * 2));
}

int enqueue_step(rbd_ctx_t ctx, const LoopBufs& L) {
  DevState* st = ptr<DevState>(ctx->state);
  ExtBufs b{};
  b.B = L.Y;
  b.m = L.m;
  b.dcap = L.d_max;
  b.X = L.X;
  b.ldx = L.ldx;
  b.c = ptr<double>(ctx->c);
  b.w = ptr<double>(ctx->w);
  b.p = ptr<double>(ctx->p);
  b.nrm = ptr<double>(ctx->nrm);
  b.partial = ptr<double>(ctx->partial);
  b.ybase = L.Y;
  b.use_d = 1;
  b.selected = ptr<long long>(ctx->sel);
  b.st = st;
  TRY(enqueue_extension(ctx, b));

  const int vec = (L.ldx % 2 == 0 && L.m % 2 == 0 && aligned16(L.X) && aligned16(L.Y)) ? 2 : 1;
  SweepArgs s{};
  s.A = L.X;
  s.lda = L.ldx;
  s.m = L.m;
  s.ncols = L.n;
  s.vbase = L.Y;
  s.vstride = L.m;
  s.vsel = 1;
  s.partial = ptr<double>(ctx->partial);
  s.pstride = L.n;
  s.st = st;
  s.gate = GATE_LIVE;
  TRY(launch_sweep(ctx, s, vec, MODE_DOT, true, L.n));

  FinalizeArgs f{};
  f.partial = ptr<double>(ctx->partial);
  f.S = cdiv(L.m, kChunk);
  f.n = L.n;
  f.T = L.T;
  f.r = ptr<double>(ctx->resid);
  f.col_sq = ptr<double>(ctx->colsq);
  f.st = st;
  f.rec = ptr<Rec>(ctx->rec);
  f.counter = ptr<unsigned>(ctx->counter);
  f.history = ptr<double>(ctx->hist);
  f.cbuf = ptr<double>(ctx->c);
  f.mode = 0;
  k_finalize<<<finalize_grid(ctx, L.n), kThreads, 0, ctx->stream>>>(f);
  ctx->launches++;
  CU(cudaGetLastError());
  return RBD_OK;
}

// One greedy step with a diagonal weight (rbd_weighted.cuh): extension (K4,
// Euclidean, unchanged), a o xi, the YAY row over Y, one X pass for the T and
// YAX rows, and the weighted finalize/argmax.
int enqueue_step_diag(rbd_ctx_t ctx, const LoopBufs& L, const double* diag) {
  DevState* st = ptr<DevState>(ctx->state);
  ExtBufs b{};
  b.B = L.Y;
  b.m = L.m;
  b.dcap = L.d_max;
  b.X = L.X;
  b.ldx = L.ldx;
  b.c = ptr<double>(ctx->c);
  b.w = ptr<double>(ctx->w);
  b.p = ptr<double>(ctx->p);
  b.nrm = ptr<double>(ctx->nrm);
  b.partial = ptr<double>(ctx->partial);
  b.ybase = L.Y;
  b.use_d = 1;
  b.selected = ptr<long long>(ctx->sel);
  b.st = st;
  TRY(enqueue_extension(ctx, b));
  const int gv = diag_vec_grid(ctx, L.m);
  k_diag_vec<<<gv, kThreads, 0, ctx->stream>>>(L.Y, L.m, diag, ptr<double>(ctx->wd_axi),
                                               ptr<double>(ctx->wd_yy), st);
  ctx->launches++;
  // YAY[d, 0:d] = Y' (a o xi): chunked dots over the first st->d columns of Y
  const int vy = (L.m % 2 == 0 && aligned16(L.Y) && aligned16(ctx->wd_axi.p)) ? 2 : 1;
  SweepArgs s{};
  s.A = L.Y;
  s.lda = L.m;
  s.m = L.m;
  s.ncols = L.d_max;
  s.v = ptr<double>(ctx->wd_axi);
  s.partial = ptr<double>(ctx->ppart);
  s.pstride = L.d_max;
  s.st = st;
  s.gate = GATE_LIVE;
  s.csel = 1;
  TRY(launch_sweep(ctx, s, vy, MODE_DOT, false, L.d_max));
  k_coef_combine<<<(unsigned)std::max<long long>(1, cdiv(L.d_max, 256)), 256, 0, ctx->stream>>>(
      ptr<double>(ctx->ppart), cdiv(L.m, kChunk), L.d_max, ptr<double>(ctx->wd_yrow), st, GATE_LIVE);
  ctx->launches++;
  // T and YAX rows in one X pass
  const int vx = (L.ldx % 2 == 0 && L.m % 2 == 0 && aligned16(L.X) && aligned16(L.Y) &&
                  aligned16(ctx->wd_axi.p)) ? 2 : 1;
  const long long ntiles = cdiv(L.m, kChunk) * cdiv(L.n, kCols);
  const int gx = (int)std::max<long long>(1, std::min<long long>(ntiles, (long long)ctx->nsm * 2));
  if (vx == 2)
    k_sweep_diag<2><<<gx, kThreads, 0, ctx->stream>>>(L.X, L.ldx, L.m, L.n, L.Y,
                                                      ptr<double>(ctx->wd_axi),
                                                      ptr<double>(ctx->partial),
                                                      ptr<double>(ctx->wd_part2), st);
  else
    k_sweep_diag<1><<<gx, kThreads, 0, ctx->stream>>>(L.X, L.ldx, L.m, L.n, L.Y,
                                                      ptr<double>(ctx->wd_axi),
                                                      ptr<double>(ctx->partial),
                                                      ptr<double>(ctx->wd_part2), st);
  ctx->launches++;
  FinalizeDiagArgs f{};
  f.f.partial = ptr<double>(ctx->partial);
  f.f.S = cdiv(L.m, kChunk);
  f.f.n = L.n;
  f.f.T = L.T;
  f.f.r = ptr<double>(ctx->resid);
  f.f.col_sq = ptr<double>(ctx->colsq);
  f.f.st = st;
  f.f.rec = ptr<Rec>(ctx->rec);
  f.f.counter = ptr<unsigned>(ctx->counter);
  f.f.history = ptr<double>(ctx->hist);
  f.f.cbuf = ptr<double>(ctx->c);
  f.f.mode = 0;
  f.partial2 = ptr<double>(ctx->wd_part2);
  f.YAX = ptr<double>(ctx->wd_yax);
  f.yrow = ptr<double>(ctx->wd_yrow);
  f.yy_part = ptr<double>(ctx->wd_yy);
  f.yy_np = gv;
  f.cross = ptr<double>(ctx->wd_cross);
  f.quad = ptr<double>(ctx->wd_quad);
  f.colsq_a = ptr<double>(ctx->wd_colsq);
  const int gf = (int)std::max<long long>(
      1, std::min<long long>(cdiv(L.n, kFdCols), (long long)ctx->nsm * 4));
  k_finalize_diag<<<gf, kThreads, 0, ctx->stream>>>(f);
  ctx->launches++;
  CU(cudaGetLastError());
  return RBD_OK;
}

bool use_fused(long long d_max) { return d_max <= kFMaxCoef; }

// Weighted loop: one persistent launch unless its decider's YAY matvec (d^2
// doubles per step, read by one CTA) would rival the X pass (m n doubles at
// HBM rate): d^2 <= m n / 256. RBD_DIAG_PATH=persistent|steps overrides.
bool diag_persistent(rbd_ctx_t ctx, long long d_max, long long m, long long n) {
  if (ctx->path != 0 || !use_fused(d_max)) return false;
  if (const char* e = getenv("RBD_DIAG_PATH")) {
    if (std::string(e) == "persistent") return true;
    if (std::string(e) == "steps") return false;
  }
  return (double)d_max * (double)d_max <= (double)m * (double)n / 256.0;
}

int fused_grid(rbd_ctx_t ctx, long long m) {
  return (int)std::max<long long>(1, std::min<long long>(cdiv(m, kFRows), ctx->fused_grid_cap));
}

size_t fused_smem(long long dcap) { return sizeof(double) * 3 * (size_t)std::max<long long>(dcap, 1); }
// c and p vectors, each zero-padded by one P1 batch (16 loads x kWarps columns);
// weighted: + p_k and the YAY row for the finaliser
// fold: + this CTA's share of p_k (d doubles per P1 half)
size_t persist_smem(long long dcap, bool diag, bool fold) {
  const size_t d = (size_t)std::max<long long>(dcap, 1);
  const size_t halves = RBD_FOLD_ROWS / 64;
  return sizeof(double) * (2 * (d + 16 * kWarps) + (diag ? 2 * (d + 1) + 2 : 0) + (fold ? halves * d : 0)) +
         (diag ? (size_t)kSvBytes : 0);   // DIAG: X-tile vector slots (rbd_weighted.cuh)
}

// RBD_FOLD=1: the identity loop forms p_k = Y'w1_k inside P1 (FOLD
// instantiation), so each step reads Y from HBM once instead of twice (P1 +
// the Y'w1 groups) when Y outgrows L2; steps with k above fold_kmax
// (RBD_FOLD_KMAX) keep the Y'w1 sweep, since the 296 CTAs' 64-row blocks (64 k
// doubles each) must stay L2-resident between P1's read and the fold's
// re-read (tools/microbench/p1_fold.cu).
bool use_fold(long long m, long long d_max) {
  if (const char* e = getenv("RBD_FOLD")) return atoi(e) != 0 && (double)m * (double)d_max > 0.0;
  // off by default: once the instrumentation checks left the base kernel
  // (RBD_INSTRUMENT), its C2 loop (2977 ms) beat the FOLD one (3004 ms; fp32
  // storage 1811 vs 1859 ms): the fold's P1 costs more than the second Y read
  return false;
}
long long fold_kmax(int grid) {
  if (const char* e = getenv("RBD_FOLD_KMAX")) return atoll(e);
  return (long long)(80.0e6 / (8.0 * 64.0 * std::max(grid, 1)));
}

// X tiles claimed ahead of the Y'w1 groups in every step of the fp64 identity
// loop (RBD_YDELAY overrides, in tiles): half a wave lets the first claimers
// stream X instead of waiting for the slowest CTA's P1. Measured (A/B in one
// process, tools/ab_env.py): C1 46.18 -> 45.89 ms at grid/2, 46.09 at one
// wave, 46.46 at two; C2 unchanged (2930.8 / 2931.0 / 2933.3 ms). The fp32
// loop, once its tiles lost the trailing barrier (tools/ab_arms.py --f32):
// C1 31.40 -> 31.13 ms at grid/2, 31.61 at one wave; C2 unchanged.
long long y_delay(int grid, bool xf32) {
  if (const char* e = getenv("RBD_YDELAY")) return atoll(e);
  (void)xf32;
  return grid / 2;
}

// Materialise a pending column / clear the pending flag (used after the loop).
int enqueue_fused_ext(rbd_ctx_t ctx, const LoopBufs& L) {
  DevState* st = ptr<DevState>(ctx->state);
  FusedArgs fa{};
  fa.Y = L.Y;
  fa.m = L.m;
  fa.X = L.X;
  fa.ldx = L.ldx;
  fa.c = ptr<double>(ctx->c);
  fa.p = ptr<double>(ctx->p);
  fa.w = ptr<double>(ctx->w);
  fa.ppart = ptr<double>(ctx->ppart);
  fa.pstride = L.d_max;
  fa.npart = ptr<double>(ctx->nrm);
  fa.st = st;
  fa.dcap = L.d_max;
  const int ga = fused_grid(ctx, L.m);
  k_ext_fused<<<ga, kThreads, fused_smem(L.d_max), ctx->stream>>>(fa);
  ctx->launches++;
  ReduceArgs ra{};
  ra.ppart = ptr<double>(ctx->ppart);
  ra.pstride = L.d_max;
  ra.nparts = ga;
  ra.npart = ptr<double>(ctx->nrm);
  ra.p = ptr<double>(ctx->p);
  ra.st = st;
  ra.selected = ptr<long long>(ctx->sel);
  ra.w1 = ptr<double>(ctx->w);
  ra.Y = L.Y;
  ra.m = L.m;
  k_ext_reduce<<<(unsigned)std::max<long long>(1, cdiv(L.d_max, 32)), kThreads, 0, ctx->stream>>>(ra);
  ctx->launches++;
  CU(cudaGetLastError());
  return RBD_OK;
}

// One greedy step on the fused path: A (extension pass, one Y read), B
// (reduce + reorth decision + breakdown), C (fused X sweep on w1), D
// (normalise/correct T row, residuals, argmax, state).
int enqueue_step_fused(rbd_ctx_t ctx, const LoopBufs& L) {
  DevState* st = ptr<DevState>(ctx->state);
  TRY(enqueue_fused_ext(ctx, L));
  const int vec = (L.ldx % 2 == 0 && aligned16(L.X) && aligned16(ctx->w.p)) ? 2 : 1;
  SweepArgs s{};
  s.A = L.X;
  s.lda = L.ldx;
  s.m = L.m;
  s.ncols = L.n;
  s.v = ptr<double>(ctx->w);
  s.partial = ptr<double>(ctx->partial);
  s.pstride = L.n;
  s.st = st;
  s.gate = GATE_LIVE;
  TRY(launch_sweep(ctx, s, vec, MODE_DOT, true, L.n));
  Finalize2Args f{};
  f.partial = ptr<double>(ctx->partial);
  f.S = cdiv(L.m, kChunk);
  f.n = L.n;
  f.T = L.T;
  f.p = ptr<double>(ctx->p);
  f.r = ptr<double>(ctx->resid);
  f.col_sq = ptr<double>(ctx->colsq);
  f.st = st;
  f.rec = ptr<Rec>(ctx->rec);
  f.counter = ptr<unsigned>(ctx->counter);
  f.history = ptr<double>(ctx->hist);
  f.cbuf = ptr<double>(ctx->c);
  f.mode = 0;
  const int g = (int)std::max<long long>(1, std::min<long long>(cdiv(L.n, kF2Cols), (long long)ctx->nsm * 4));
  k_finalize_fused<<<g, kThreads, 0, ctx->stream>>>(f);
  ctx->launches++;
  CU(cudaGetLastError());
  return RBD_OK;
}

int persistent_grid(rbd_ctx_t ctx, int vec, long long d_max, bool diag, bool xf32, bool fold) {
  int occ = 0;
  const size_t smem = persist_smem(d_max, diag, fold);
  if (fold)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, xf32 ? k_rbd_persistent<2, false, false, true, true> : k_rbd_persistent<2, false, false, false, true>,
        kThreads, smem);
  else if (xf32)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, vec == 2 ? k_rbd_persistent<2, false, false, true> : k_rbd_persistent<1, false, false, true>,
        kThreads, smem);
  else if (diag)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, vec == 2 ? k_rbd_persistent<2, false, true> : k_rbd_persistent<1, false, true>,
        kThreads, smem);
  else if (vec == 2)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rbd_persistent<2, false>, kThreads, smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rbd_persistent<1, false>, kThreads, smem);
  occ = std::min(occ, 2);
  return occ * ctx->nsm;
}

// The whole greedy loop in one cooperative launch (single GPU); diag != nullptr:
// the weighted loop (row f1; the caller has sized the wd_* buffers and zeroed
// cross/quad).
int launch_persistent(rbd_ctx_t ctx, const LoopBufs& L, const double* diag = nullptr) {
  const bool xf32 = L.Xf != nullptr;
  // VEC: 16-byte pairs of Y / w rows in P1 (and of X in the fp64 sweep; the
  // fp32 sweep picks float4 loads separately, so its VEC never depends on ldx)
  const bool xpairs = xf32 || (L.ldx % 2 == 0 && aligned16(L.X));
  const int vec = (xpairs && L.m % 2 == 0 && aligned16(L.Y) && aligned16(ctx->w.p) &&
                   (!diag || aligned16(ctx->wd_axi.p))) ? 2 : 1;
  const bool fold = !diag && vec == 2 && use_fold(L.m, L.d_max);
  const int grid = persistent_grid(ctx, vec, L.d_max, diag != nullptr, xf32, fold);
  if (grid < 1) return set_err(RBD_ERR_CUDA, "persistent kernel: zero occupancy");
  const long long S = cdiv(L.m, kChunk);
  const long long ngx = cdiv(L.n, kCols);
  TRY(ensure(ctx->ppart, sizeof(double) * (size_t)std::max<long long>(grid, S) * L.d_max));
  TRY(ensure(ctx->ctl, sizeof(StepCtl)));
  TRY(ensure(ctx->gcnt, sizeof(double) * 2 * (size_t)(L.d_max + 1)));   // p_k, by step parity
  TRY(ensure(ctx->ygcnt, sizeof(Rec) * (size_t)grid));                  // CTA records
  TRY(ensure(ctx->rdy, sizeof(unsigned long long) * (size_t)(S + 1)));
  CU(cudaMemsetAsync(ctx->ctl.p, 0, sizeof(StepCtl), ctx->stream));
  CU(cudaMemsetAsync(ctx->rdy.p, 0, sizeof(unsigned long long) * (size_t)(S + 1), ctx->stream));
  CU(cudaMemsetAsync(ctx->bar.p, 0, 64, ctx->stream));
  // chunk partials double as ready flags: NaN (all bytes 0xFF) = not written
  CU(cudaMemsetAsync(ctx->partial.p, 0xFF, sizeof(double) * (size_t)S * L.n, ctx->stream));
  (void)ngx;
  TRY(ensure(ctx->nrm, sizeof(double) * std::max<long long>(gemv_grid(L.m), grid)));
  TRY(ensure(ctx->rec, sizeof(Rec) * (size_t)std::max(grid, ctx->nsm * 8)));
  PersistArgs a{};
  a.X = L.X;
  a.Xf = L.Xf;
  a.xvec4 = (xf32 && L.ldx % 4 == 0 && aligned16(L.Xf)) ? 1 : 0;
  a.ldx = L.ldx;
  a.m = L.m;
  a.n = L.n;
  a.Y = L.Y;
  a.T = L.T;
  a.w = ptr<double>(ctx->w);
  a.p = ptr<double>(ctx->gcnt);
  a.ppart = ptr<double>(ctx->ppart);
  a.npart = ptr<double>(ctx->nrm);
  a.partial = ptr<double>(ctx->partial);
  a.r = ptr<double>(ctx->resid);
  a.col_sq = ptr<double>(ctx->colsq);
  a.rec = ptr<Rec>(ctx->ygcnt);
  a.history = ptr<double>(ctx->hist);
  a.selected = ptr<long long>(ctx->sel);
  a.st = ptr<DevState>(ctx->state);
  a.bar = ptr<unsigned>(ctx->bar);
  a.d_max = L.d_max;
  a.ctl = ptr<StepCtl>(ctx->ctl);
  a.rdy = ptr<unsigned long long>(ctx->rdy);
  a.forced = ctx->forced_h.empty() ? nullptr : ptr<long long>(ctx->forced);
  a.nforced = (long long)ctx->forced_h.size();
  a.ydelay = y_delay(grid, xf32);
  a.fold_kmax = fold ? fold_kmax(grid) : 0;
  if (diag) {
    TRY(ensure(ctx->wd_ppart2, sizeof(double) * (size_t)std::max<long long>(grid, S) * L.d_max));
    TRY(ensure(ctx->wd_q, sizeof(double) * (size_t)(L.d_max + 1)));
    TRY(ensure(ctx->wd_yay, sizeof(double) * (size_t)L.d_max * (size_t)L.d_max));
    TRY(ensure(ctx->wd_yy, sizeof(double) * (size_t)std::max<long long>(grid, diag_vec_grid(ctx, L.m))));
    CU(cudaMemsetAsync(ctx->wd_part2.p, 0xFF, sizeof(double) * (size_t)S * L.n, ctx->stream));
    a.diag = diag;
    a.aw = ptr<double>(ctx->wd_axi);
    a.npart2 = ptr<double>(ctx->wd_yy);
    a.ppart2 = ptr<double>(ctx->wd_ppart2);
    TRY(ensure(ctx->wd_yslice, sizeof(double) * 2 * (size_t)(L.d_max / kYSlice + 2)));
    a.yslice = ptr<double>(ctx->wd_yslice);
    a.q = ptr<double>(ctx->wd_q);
    a.partial2 = ptr<double>(ctx->wd_part2);
    a.YAX = ptr<double>(ctx->wd_yax);
    a.YAY = ptr<double>(ctx->wd_yay);
    a.yrow = ptr<double>(ctx->wd_yrow);
    a.cross = ptr<double>(ctx->wd_cross);
    a.quad = ptr<double>(ctx->wd_quad);
    a.colsq_a = ptr<double>(ctx->wd_colsq);
  }
  a.progress = (ctx->ystream_dst && ctx->d_progress) ? ctx->d_progress : nullptr;
  if (a.progress) *(volatile long long*)ctx->h_progress = 0;
  a.phase_ns = nullptr;
  if ((getenv("RBD_PHASE_TIMING") || getenv("RBD_TRACE_STEP")) && !RBD_INSTRUMENT) {
    static bool warned = false;
    if (!warned) fprintf(stderr, "[rbd] RBD_PHASE_TIMING / RBD_TRACE_STEP need a build with "
                                 "RBD_NVCC_DEFS=-DRBD_INSTRUMENT=1; ignored\n");
    warned = true;
  }
  if (RBD_INSTRUMENT && getenv("RBD_PHASE_TIMING")) {
    TRY(ensure(ctx->scratch1, 256));
    cudaMemsetAsync(ctx->scratch1.p, 0, 128, ctx->stream);
    a.phase_ns = ptr<unsigned long long>(ctx->scratch1);
  }
  a.trace = nullptr;
  DevBuf tracebuf;
  if (const char* ts = RBD_INSTRUMENT ? getenv("RBD_TRACE_STEP") : nullptr) {
    TRY(ensure(tracebuf, sizeof(unsigned long long) * (size_t)grid * kTraceWords));
    cudaMemsetAsync(tracebuf.p, 0, sizeof(unsigned long long) * (size_t)grid * kTraceWords, ctx->stream);
    a.trace = ptr<unsigned long long>(tracebuf);
    a.trace_step = atoll(ts);
  }
  void* args[] = {&a};
  const size_t smem = persist_smem(L.d_max, diag != nullptr, fold);
  void* fn = fold ? (xf32 ? (void*)k_rbd_persistent<2, false, false, true, true>
                          : (void*)k_rbd_persistent<2, false, false, false, true>)
             : xf32 ? (vec == 2 ? (void*)k_rbd_persistent<2, false, false, true>
                              : (void*)k_rbd_persistent<1, false, false, true>)
             : diag ? (vec == 2 ? (void*)k_rbd_persistent<2, false, true>
                              : (void*)k_rbd_persistent<1, false, true>)
                  : (vec == 2 ? (void*)k_rbd_persistent<2, false> : (void*)k_rbd_persistent<1, false>);
  if (getenv("RBD_DEBUG_LAUNCH"))
    fprintf(stderr, "[launch] persistent vec=%d fold=%d diag=%d xf32=%d grid=%d smem=%zu fold_kmax=%lld\n", vec,
            (int)fold, diag != nullptr, (int)xf32, grid, smem, a.fold_kmax);
  cudaError_t e = cudaLaunchCooperativeKernel(fn, grid, kThreads, args, smem, ctx->stream);
  ctx->launches++;
  if (e != cudaSuccess)
    return set_err(RBD_ERR_CUDA, std::string("persistent launch: ") + cudaGetErrorString(e));
  if (a.trace) {
    std::vector<unsigned long long> h((size_t)grid * kTraceWords);
    cudaMemcpyAsync(h.data(), a.trace, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost,
                    ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    const char* path = getenv("RBD_TRACE_FILE");
    FILE* f = fopen(path ? path : "rbd_trace.bin", "wb");
    if (f) {
      fwrite(&grid, sizeof(int), 1, f);
      fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
      fclose(f);
    }
    release(tracebuf);
  }
  if (a.phase_ns) {
    unsigned long long h[10];
    cudaMemcpyAsync(h, a.phase_ns, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    const char* nm[10] = {"P1 ext", "bar1", "P2 queue", "bar2", "state", "claim wait",
                          "Y tiles", "X tiles", "fin spin", "fin/other"};
    for (int i = 0; i < 10; ++i) fprintf(stderr, "[phase] %-16s %10.3f ms\n", nm[i], h[i] / 1e6);
  }
  return RBD_OK;
}

int ensure_loop_buffers(rbd_ctx_t ctx, long long m, long long n, long long d_max) {
  const long long S = cdiv(m, kChunk);
  TRY(ensure(ctx->partial, sizeof(double) * S * std::max(n, d_max)));
  TRY(ensure(ctx->rec, sizeof(Rec) * (size_t)ctx->nsm * 8));
  TRY(ensure(ctx->counter, 64));
  TRY(ensure(ctx->state, sizeof(DevState)));
  TRY(ensure(ctx->colsq, sizeof(double) * n));
  TRY(ensure(ctx->resid, sizeof(double) * n));
  TRY(ensure(ctx->w, sizeof(double) * m));
  TRY(ensure(ctx->c, sizeof(double) * (d_max + 1)));
  TRY(ensure(ctx->p, sizeof(double) * (d_max + 1)));
  TRY(ensure(ctx->nrm, sizeof(double) * gemv_grid(m)));
  TRY(ensure(ctx->hist, sizeof(double) * d_max));
  TRY(ensure(ctx->sel, sizeof(long long) * d_max));
  TRY(ensure(ctx->out_rec, sizeof(Rec) * 16));
  TRY(ensure(ctx->ppart, sizeof(double) * (size_t)ctx->fused_grid_cap * d_max));
  TRY(ensure(ctx->nrm, sizeof(double) * std::max<long long>(gemv_grid(m), ctx->fused_grid_cap)));
  return RBD_OK;
}

constexpr int kGraphSteps = 8;

int get_step_graph(rbd_ctx_t ctx, const LoopBufs& L) {
  GraphKey k;
  k.X = L.X;
  k.Y = L.Y;
  k.T = L.T;
  k.m = L.m;
  k.n = L.n;
  k.ldx = L.ldx;
  k.d_max = L.d_max;
  k.stream = ctx->stream;
  k.steps = kGraphSteps;
  DevBuf* bl[8] = {&ctx->partial, &ctx->rec, &ctx->state, &ctx->colsq,
                   &ctx->resid,   &ctx->w,   &ctx->c,     &ctx->ppart};
  for (int i = 0; i < 8; ++i) k.bufs[i] = bl[i]->p;
  if (ctx->gexec && ctx->gkey == k) return RBD_OK;
  if (ctx->gexec) {
    cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
  }
  const long long before = ctx->launches;
  CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  int rc = RBD_OK;
  for (int s = 0; s < kGraphSteps && rc == RBD_OK; ++s)
    rc = use_fused(L.d_max) ? enqueue_step_fused(ctx, L) : enqueue_step(ctx, L);
  cudaGraph_t g = nullptr;
  cudaError_t ec = cudaStreamEndCapture(ctx->stream, &g);
  ctx->launches = before;  // captured launches are counted per replay
  if (rc != RBD_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (ec != cudaSuccess) return set_err(RBD_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
  size_t nn = 0;
  cudaGraphGetNodes(g, nullptr, &nn);
  ctx->graph_nodes = (long long)nn;
  cudaError_t ei = cudaGraphInstantiate(&ctx->gexec, g, 0);
  cudaGraphDestroy(g);
  if (ei != cudaSuccess) return set_err(RBD_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei));
  ctx->gkey = k;
  return RBD_OK;
}

// Validation shared by the single- and multi-GPU entries: reference order of
// decompose.cpp:56-64 after the K1 flags are known.
int validate_after_init(const rbd_config_t* cfg, long long m, long long n, const DevState& hs,
                        bool diag_supplied, double diag_max) {
  if (hs.flags_nonfinite)
    return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: matrix has non-finite entries");
  if (cfg->d_max < 1 || cfg->d_max > n)
    return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: d_max must satisfy 1 <= d_max <= n");
  if (!(cfg->eps_R >= 0.0)) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: eps_R must be >= 0");
  if (cfg->weight_kind != RBD_WEIGHT_IDENTITY) {
    if (cfg->weight_dim != 0 && cfg->weight_dim != m)
      return set_err(RBD_ERR_INCOMPATIBLE_WEIGHT, "decompose: weight dimension != m");
    if (!(cfg->weight_kind == RBD_WEIGHT_DIAGONAL && diag_supplied))
      return set_err(RBD_ERR_INVALID_ARGUMENT,
                     cfg->weight_kind == RBD_WEIGHT_DIAGONAL
                         ? "decompose: a diagonal weight runs through rbd_decompose_diag_*"
                         : "decompose: sparse SPD weights are out of scope on the B200 path "
                           "(SURVEY.md §8(f1))");
  }
  if (!hs.flags_nonzero)
    return set_err(RBD_ERR_DEGENERATE_INPUT, "decompose: zero matrix, no basis can be built");
  // A finite X whose largest column norm overflows (entries beyond ~1e154):
  // in the reference max_col_norm = inf makes breakdown_tol = inf
  // (decompose.cpp:70-74), so the first mgs_project breaks down and the call
  // ends in DegenerateInput (:104-105). Stop here with that outcome: the
  // device loop would otherwise meet inf - inf = NaN dot products, and its
  // chunk partials use NaN to mean "not written yet".
  double max_colsq;
  std::memcpy(&max_colsq, &hs.max_colsq_bits, sizeof(double));
  if (!std::isfinite(max_colsq))
    return set_err(RBD_ERR_DEGENERATE_INPUT,
                   "decompose: start column is numerically zero, no basis built "
                   "(max column norm overflows, breakdown tolerance is inf)");
  // Weighted sums a_i x_ij y_i (workspace.cpp:24-29,61-79) stay finite when
  // max_i a_i * max_j ||x_j||^2 does (Cauchy-Schwarz with ||y|| <= ||x||).
  if (diag_max > 0.0 && !std::isfinite(diag_max * max_colsq))
    return set_err(RBD_ERR_INVALID_ARGUMENT,
                   "decompose: weighted column norms overflow (max a_i * max ||x_j||^2 is not finite)");
  return RBD_OK;
}

int start_column(const rbd_config_t* cfg, long long n, long long* out) {
  // decompose.cpp:37-49
  if (cfg->start_kind == RBD_START_FIXED_COLUMN) {
    if (cfg->start_column < 0 || cfg->start_column >= n)
      return set_err(RBD_ERR_INDEX_OUT_OF_RANGE, "start column index out of range");
    *out = cfg->start_column;
  } else {
    std::mt19937_64 rng(cfg->start_seed);
    *out = (long long)std::uniform_int_distribution<long>(0, (long)n - 1)(rng);
  }
  return RBD_OK;
}

double breakdown_tolerance(const rbd_config_t* cfg, long long m, double max_colsq) {
  // decompose.cpp:70-74
  const double max_col_norm = std::sqrt(max_colsq);
  const double noise_floor = max_col_norm * std::sqrt(static_cast<double>(m)) *
                             std::numeric_limits<double>::epsilon() * 16.0;
  return std::max(cfg->breakdown_tol < 0.0 ? cfg->eps_R : cfg->breakdown_tol, noise_floor);
}

// diagonal weight values: positive and finite (weight.cpp:11-17)
int check_diagonal(const double* h, int64_t len) {
  if (len <= 0) return set_err(RBD_ERR_INVALID_ARGUMENT, "diagonal weight must be non-empty");
  for (int64_t i = 0; i < len; ++i)
    if (!(h[i] > 0.0) || !std::isfinite(h[i]))
      return set_err(RBD_ERR_INVALID_ARGUMENT,
                     "diagonal weight entries must be strictly positive and finite");
  return RBD_OK;
}

}  // namespace rbdc

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* rbd_last_error(void) { return g_err.c_str(); }

// for the library's other translation units (csrc/rbd_internal.h)
__attribute__((visibility("hidden"))) int rbd_internal_set_error(int code, const char* msg) {
  g_err = msg;
  return code;
}
int rbd_abi_version(void) { return RBD_ABI_VERSION; }

void rbd_config_default(rbd_config_t* cfg) {
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->d_max = 1;             // decompose.hpp:26
  cfg->eps_R = 0.0;           // :27
  cfg->start_kind = RBD_START_FIXED_COLUMN;
  cfg->start_column = 0;      // :28
  cfg->reorthogonalize = 0;   // :30
  cfg->breakdown_tol = -1.0;  // :35
  cfg->weight_kind = RBD_WEIGHT_IDENTITY;
}

int rbd_ctx_create(int device, rbd_ctx_t* out) {
  if (!out) return set_err(RBD_ERR_INVALID_ARGUMENT, "rbd_ctx_create: null output");
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    return set_err(RBD_ERR_INVALID_ARGUMENT, "rbd_ctx_create: no such CUDA device");
  CU(cudaSetDevice(device));
  auto* ctx = new rbd_ctx_s();
  ctx->device = device;
  cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return set_err(RBD_ERR_CUDA, std::string("stream create: ") + cudaGetErrorString(e));
  }
  ctx->stream = ctx->own_stream;
  cudaMallocHost(&ctx->h_state, sizeof(DevState));
  cudaMallocHost(&ctx->h_rec, sizeof(Rec) * 4);
  if (cudaHostAlloc(&ctx->h_progress, sizeof(long long), cudaHostAllocMapped) == cudaSuccess) {
    if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->d_progress), ctx->h_progress, 0) !=
        cudaSuccess) {
      cudaGetLastError();
      ctx->d_progress = nullptr;
    }
  } else {
    cudaGetLastError();
    ctx->h_progress = nullptr;
  }
  int o = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_sweep<2, MODE_DOT, true>, kThreads, 0) ==
          cudaSuccess && o > 0)
    ctx->occ_sweep2 = o;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_sweep<1, MODE_DOT, true>, kThreads, 0) ==
          cudaSuccess && o > 0)
    ctx->occ_sweep1 = o;
  cudaFuncSetAttribute(k_ext_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)fused_smem(kFMaxCoef));
  ctx->fused_grid_cap = 2 * ctx->nsm;
  {
    const int sm_id = (int)persist_smem(kFMaxCoef, false);
    const int sm_sh = sm_id;
    const int sm_f32 = sm_id;
    cudaFuncSetAttribute(k_rbd_persistent<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_id);
    cudaFuncSetAttribute(k_rbd_persistent<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_id);
    cudaFuncSetAttribute(k_rbd_persistent<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_sh);
    cudaFuncSetAttribute(k_rbd_persistent<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_sh);
    cudaFuncSetAttribute(k_rbd_persistent<2, false, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm_f32);
    cudaFuncSetAttribute(k_rbd_persistent<1, false, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm_f32);
    cudaFuncSetAttribute(k_rbd_persistent<2, false, false, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)persist_smem(kFMaxCoef, false, true));
    cudaFuncSetAttribute(k_rbd_persistent<2, false, false, true, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)persist_smem(kFMaxCoef, false, true));
  }
  cudaFuncSetAttribute(k_rbd_persistent<2, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)persist_smem(kFMaxCoef, true));
  cudaFuncSetAttribute(k_rbd_persistent<1, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)persist_smem(kFMaxCoef, true));
  if (const char* pth = getenv("RBD_PATH")) ctx->path = (std::string(pth) == "graph") ? 1 : 0;
  if (ensure(ctx->bar, 64) == RBD_OK) cudaMemset(ctx->bar.p, 0, 64);
  *out = ctx;
  return RBD_OK;
}

int rbd_ctx_destroy(rbd_ctx_t ctx) {
  if (!ctx) return RBD_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (rbd_ctx_t sub : ctx->virt) rbd_ctx_destroy(sub);
  ctx->virt.clear();
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  DevBuf* bl[] = {&ctx->partial, &ctx->rec,  &ctx->counter, &ctx->state, &ctx->colsq,
                  &ctx->resid,   &ctx->w,    &ctx->c,       &ctx->p,     &ctx->nrm,
                  &ctx->hist,    &ctx->sel,  &ctx->out_rec, &ctx->scratch1,
                  &ctx->hX,      &ctx->hX2,  &ctx->hY,      &ctx->hT,    &ctx->ppart, &ctx->bar,
                  &ctx->wd_axi,  &ctx->wd_yy, &ctx->wd_part2, &ctx->wd_yrow, &ctx->wd_yax,
                  &ctx->wd_cross, &ctx->wd_quad, &ctx->wd_colsq, &ctx->wd_diag,
                  &ctx->wd_ppart2, &ctx->wd_q, &ctx->wd_yay, &ctx->wd_yslice, &ctx->forced,
                  &ctx->nn_part, &ctx->nn_coords, &ctx->pj_ws,
                  &ctx->ctl,     &ctx->gcnt, &ctx->ygcnt,   &ctx->rdy,   &ctx->send,  &ctx->recv,
                  &ctx->srec,    &ctx->rrec,
                  &ctx->hs[0],   &ctx->hs[1], &ctx->hs[2],  &ctx->hs[3], &ctx->hs[4],
                  &ctx->pm_X[0], &ctx->pm_X[1], &ctx->pm_T[0], &ctx->pm_T[1], &ctx->pm_E[0],
                  &ctx->pm_E[1]};
  for (DevBuf* b : bl) release(*b);
  if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
  if (ctx->h_done) cudaFreeHost(ctx->h_done);
  if (ctx->h_state) cudaFreeHost(ctx->h_state);
  if (ctx->h_progress) cudaFreeHost(ctx->h_progress);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->up_stream) cudaStreamDestroy(ctx->up_stream);
  if (ctx->h_rec) cudaFreeHost(ctx->h_rec);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  rbd_comm_release(ctx);
  delete ctx;
  return RBD_OK;
}

int rbd_ctx_set_stream(rbd_ctx_t ctx, void* s) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
  return RBD_OK;
}

int64_t rbd_ctx_launch_count(rbd_ctx_t ctx) { return ctx ? ctx->launches : 0; }

int rbd_set_forced_selection(rbd_ctx_t ctx, const int64_t* h_selected, int64_t count) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "forced selection: null context");
  if (count < 0 || (count > 0 && !h_selected))
    return set_err(RBD_ERR_INVALID_ARGUMENT, "forced selection: bad sequence");
  CU(cudaSetDevice(ctx->device));
  ctx->forced_h.assign(h_selected, h_selected + count);
  if (count > 0) {
    TRY(ensure(ctx->forced, sizeof(long long) * (size_t)count));
    CU(cudaMemcpyAsync(ctx->forced.p, ctx->forced_h.data(), sizeof(long long) * (size_t)count,
                       cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  return RBD_OK;
}

int rbd_ctx_synchronize(rbd_ctx_t ctx) {
  CU(cudaStreamSynchronize(ctx->stream));
  return RBD_OK;
}

void* rbd_ctx_stream(rbd_ctx_t ctx) { return ctx ? (void*)ctx->stream : nullptr; }

namespace {
// Single-GPU decompose; diag == nullptr: identity weight (persistent loop),
// else the diagonal-weight loop of rbd_weighted.cuh (diag: m device doubles,
// already validated as a WeightSpec::diagonal).
int decompose_device_impl(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx,
                          const rbd_config_t* cfg, const double* diag, double* dY, double* dT,
                          int64_t* h_selected, double* h_history, rbd_result_t* result,
                          const float* dXf = nullptr, double diag_max = 0.0) {
  if (!ctx || !cfg) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: null context/config");
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: matrix must be non-empty");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "decompose: ldx < m");
  CU(cudaSetDevice(ctx->device));
  if (dXf) {   // fp32 storage mode runs on the persistent identity loop only
    if (cfg->weight_kind != RBD_WEIGHT_IDENTITY)
      return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: fp32 storage mode supports the identity weight only");
    if (!(ctx->path == 0 && use_fused(cfg->d_max)))
      return set_err(RBD_ERR_INVALID_ARGUMENT,
                     "decompose: fp32 storage mode runs on the persistent loop (d_max <= 4096)");
  }
  const long long d_cap = std::max<long long>(1, std::min<long long>(cfg->d_max, n));
  NvtxRange nv_all("rbd.decompose");
  TRY(ensure_loop_buffers(ctx, m, n, d_cap));
  DevState* st = ptr<DevState>(ctx->state);

  const long long launches0 = ctx->launches;
  cudaEvent_t ev0, ev1, ev2;
  CU(cudaEventCreate(&ev0));
  CU(cudaEventCreate(&ev1));
  CU(cudaEventCreate(&ev2));
  struct EvGuard {
    cudaEvent_t a, b, c;
    ~EvGuard() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      cudaEventDestroy(c);
    }
  } evg{ev0, ev1, ev2};
  // ---- K1 ----
  NvtxRange nv_k1("rbd.init (K1: validation, workspace_init)");
  CU(cudaMemsetAsync(st, 0, sizeof(DevState), ctx->stream));
  CU(cudaEventRecord(ev0, ctx->stream));
  if (dXf)
    TRY(enqueue_init_f32(ctx, dXf, m, n, ldx, ptr<double>(ctx->partial), ptr<double>(ctx->colsq),
                         ptr<double>(ctx->resid), st));
  else
    TRY(enqueue_init(ctx, dX, m, n, ldx, ptr<double>(ctx->partial), ptr<double>(ctx->colsq),
                     ptr<double>(ctx->resid), st));
  if (diag) {   // workspace_init, diagonal kind (workspace.cpp:24-29)
    TRY(ensure(ctx->wd_colsq, sizeof(double) * n));
    const int g = (int)std::max<long long>(1, std::min<long long>(n, (long long)ctx->nsm * 8));
    k_colsq_diag<<<g, kThreads, 0, ctx->stream>>>(dX, ldx, m, n, diag, ptr<double>(ctx->wd_colsq));
    ctx->launches++;
  }
  CU(cudaEventRecord(ev1, ctx->stream));
  CU(cudaMemsetAsync(ctx->counter.p, 0, 64, ctx->stream));
  CU(cudaMemcpyAsync(ctx->h_state, st, sizeof(DevState), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  nv_k1.end();
  DevState hs = *ctx->h_state;
  double init_ms = 0.0;
  {
    float t = 0.f;
    cudaEventElapsedTime(&t, ev0, ev1);
    init_ms = t;
  }
  TRY(validate_after_init(cfg, m, n, hs, diag != nullptr, diag ? diag_max : 0.0));
  double max_colsq;
  {
    unsigned long long b = hs.max_colsq_bits;
    std::memcpy(&max_colsq, &b, sizeof(double));
  }
  const double tol = breakdown_tolerance(cfg, m, max_colsq);
  long long j0 = 0;
  TRY(start_column(cfg, n, &j0));
  if (!ctx->forced_h.empty()) {   // parity re-run on a given selection sequence
    for (long long v : ctx->forced_h)
      if (v < 0 || v >= n) return set_err(RBD_ERR_INDEX_OUT_OF_RANGE, "forced selection index out of range");
    const bool pers = diag ? diag_persistent(ctx, cfg->d_max, m, n)
                           : (ctx->path == 0 && use_fused(cfg->d_max));
    if (!pers)
      return set_err(RBD_ERR_INVALID_ARGUMENT,
                     "forced selection is implemented on the persistent loop only");
    j0 = ctx->forced_h[0];
  }

  // ---- loop state ----
  hs.d = 0;
  hs.jstar = j0;
  hs.jlocal = j0;
  hs.d_max = cfg->d_max;
  hs.e_cur = std::numeric_limits<double>::infinity();
  hs.eps_R = cfg->eps_R;
  hs.breakdown_tol = tol;
  hs.done = !(0 < cfg->d_max && hs.e_cur > cfg->eps_R) ? 1 : 0;
  hs.breakdown = 0;
  hs.reorth = 0;
  hs.cfg_reorth = cfg->reorthogonalize ? 1 : 0;
  *ctx->h_state = hs;
  CU(cudaMemcpyAsync(st, ctx->h_state, sizeof(DevState), cudaMemcpyHostToDevice, ctx->stream));

  LoopBufs L{dX, m, n, ldx, cfg->d_max, dY, dT, dXf};
  NvtxRange nv_loop("rbd.loop (greedy steps)");
  if (diag) {
    const long long S = cdiv(m, kChunk);
    TRY(ensure(ctx->wd_axi, sizeof(double) * m));
    TRY(ensure(ctx->wd_yy, sizeof(double) * diag_vec_grid(ctx, m)));
    TRY(ensure(ctx->wd_part2, sizeof(double) * S * n));
    TRY(ensure(ctx->wd_yrow, sizeof(double) * d_cap));
    TRY(ensure(ctx->wd_yax, sizeof(double) * d_cap * n));
    TRY(ensure(ctx->wd_cross, sizeof(double) * n));
    TRY(ensure(ctx->wd_quad, sizeof(double) * n));
    TRY(ensure(ctx->ppart, sizeof(double) * S * d_cap));
    CU(cudaMemsetAsync(ctx->wd_cross.p, 0, sizeof(double) * n, ctx->stream));
    CU(cudaMemsetAsync(ctx->wd_quad.p, 0, sizeof(double) * n, ctx->stream));
  }
  const bool diag_pers = diag && diag_persistent(ctx, cfg->d_max, m, n);
  if (diag_pers) {   // the weighted loop in one persistent launch
    CU(cudaEventRecord(ev1, ctx->stream));
    TRY(launch_persistent(ctx, L, diag));
  } else if (diag) {
    CU(cudaEventRecord(ev1, ctx->stream));
    // host-driven steps; the done flag is polled every kDiagPoll steps, one
    // batch behind, so the device never waits for the host
    constexpr long long kDiagPoll = 8;
    volatile int* hdone = &ctx->h_state->done;
    bool pending = false;
    cudaEvent_t ev;
    CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    int rc = RBD_OK;
    for (long long step = 0; step < cfg->d_max && rc == RBD_OK; ++step) {
      rc = enqueue_step_diag(ctx, L, diag);
      if (rc != RBD_OK) break;
      if ((step + 1) % kDiagPoll == 0) {
        if (pending) {
          cudaEventSynchronize(ev);
          if (*hdone) break;
        }
        cudaMemcpyAsync((void*)&ctx->h_state->done, &st->done, sizeof(int), cudaMemcpyDeviceToHost,
                        ctx->stream);
        cudaEventRecord(ev, ctx->stream);
        pending = true;
      }
    }
    cudaEventDestroy(ev);
    if (rc != RBD_OK) return rc;
  } else if (ctx->path == 0 && use_fused(cfg->d_max)) {
    CU(cudaEventRecord(ev1, ctx->stream));
    TRY(launch_persistent(ctx, L));
  } else {
    TRY(get_step_graph(ctx, L));
    CU(cudaEventRecord(ev1, ctx->stream));
    // Replay G-step graphs; the done flag is polled one graph behind so the
    // device never waits for the host.
    volatile int* hdone = &ctx->h_state->done;
    long long launched = 0;
    bool pending = false;
    cudaEvent_t ev;
    CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    int rc = RBD_OK;
    while (launched < cfg->d_max) {
      cudaError_t e = cudaGraphLaunch(ctx->gexec, ctx->stream);
      if (e != cudaSuccess) {
        rc = set_err(RBD_ERR_CUDA, std::string("graph launch: ") + cudaGetErrorString(e));
        break;
      }
      ctx->launches += ctx->graph_nodes;
      launched += kGraphSteps;
      if (pending) {
        cudaEventSynchronize(ev);
        if (*hdone) break;
      }
      cudaMemcpyAsync((void*)&ctx->h_state->done, &st->done, sizeof(int), cudaMemcpyDeviceToHost,
                      ctx->stream);
      cudaEventRecord(ev, ctx->stream);
      pending = true;
    }
    cudaEventDestroy(ev);
    if (rc != RBD_OK) return rc;
    if (use_fused(cfg->d_max)) TRY(enqueue_fused_ext(ctx, L));  // last column's second pass
  }
  CU(cudaEventRecord(ev2, ctx->stream));
  ctx->ystream_copied = 0;
  if (ctx->ystream_dst && ctx->d_progress && ctx->path == 0 && use_fused(cfg->d_max) &&
      (!diag || diag_pers)) {
    // stream finished Y columns to the host while the loop runs (copy engine,
    // second stream), 16 columns or more per copy
    if (!ctx->copy_stream) CU(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    long long copied = 0;
    while (cudaEventQuery(ev2) == cudaErrorNotReady) {
      const long long done_cols = *(volatile long long*)ctx->h_progress;
      if (done_cols - copied >= 16) {   // Y columns and T rows [copied, done_cols)
        CU(cudaMemcpyAsync(ctx->ystream_dst + copied * m, dY + copied * m,
                           sizeof(double) * (size_t)((done_cols - copied) * m),
                           cudaMemcpyDeviceToHost, ctx->copy_stream));
        if (ctx->tstream_dst)
          CU(cudaMemcpyAsync(ctx->tstream_dst + copied * n, dT + copied * n,
                             sizeof(double) * (size_t)((done_cols - copied) * n),
                             cudaMemcpyDeviceToHost, ctx->copy_stream));
        copied = done_cols;
      }
    }
    ctx->ystream_copied = copied;
  }
  CU(cudaMemcpyAsync(ctx->h_state, st, sizeof(DevState), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  hs = *ctx->h_state;
  const long long d = hs.d;
  if (d == 0)
    return set_err(RBD_ERR_DEGENERATE_INPUT,
                   "decompose: start column is numerically zero, no basis built");
  if (h_selected)
    CU(cudaMemcpyAsync(h_selected, ctx->sel.p, sizeof(long long) * d, cudaMemcpyDeviceToHost, ctx->stream));
  if (h_history)
    CU(cudaMemcpyAsync(h_history, ctx->hist.p, sizeof(double) * d, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (result) {
    float t_loop = 0.f;
    cudaEventElapsedTime(&t_loop, ev1, ev2);
    result->d = d;
    result->breakdown = hs.breakdown;
    result->breakdown_tol = tol;
    result->max_col_norm = std::sqrt(max_colsq);
    result->init_ms = init_ms;
    result->loop_ms = t_loop;
    result->launches = ctx->launches - launches0;
  }
  return RBD_OK;
}

// WeightSpec::diagonal validation (weight.cpp:11-17) on host values.
}  // namespace

int rbd_decompose_device(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx,
                         const rbd_config_t* cfg, double* dY, double* dT, int64_t* h_selected,
                         double* h_history, rbd_result_t* result) {
  return decompose_device_impl(ctx, dX, m, n, ldx, cfg, nullptr, dY, dT, h_selected, h_history,
                               result);
}

int rbd_decompose_device_f32(rbd_ctx_t ctx, const float* dX, int64_t m, int64_t n, int64_t ldx,
                             const rbd_config_t* cfg, double* dY, double* dT, int64_t* h_selected,
                             double* h_history, rbd_result_t* result) {
  if (!dX) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: null X");
  return decompose_device_impl(ctx, nullptr, m, n, ldx, cfg, nullptr, dY, dT, h_selected, h_history,
                               result, dX);
}

int rbd_decompose_diag_device(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx,
                              const rbd_config_t* cfg, const double* d_diag, int64_t diag_len,
                              double* dY, double* dT, int64_t* h_selected, double* h_history,
                              rbd_result_t* result) {
  if (!ctx || !cfg) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: null context/config");
  if (diag_len > 0 && !d_diag) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: null diagonal");
  CU(cudaSetDevice(ctx->device));
  std::vector<double> h((size_t)std::max<int64_t>(diag_len, 0));
  if (diag_len > 0) {   // on the context stream: d_diag may have been uploaded there
    CU(cudaMemcpyAsync(h.data(), d_diag, sizeof(double) * diag_len, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  TRY(check_diagonal(h.data(), diag_len));
  rbd_config_t c = *cfg;
  c.weight_kind = RBD_WEIGHT_DIAGONAL;
  c.weight_dim = diag_len;
  if (diag_len != m) {   // decompose.cpp:61-62 order: checked after init, before the zero test
    return decompose_device_impl(ctx, dX, m, n, ldx, &c, nullptr, dY, dT, h_selected, h_history,
                                 result);
  }
  const double diag_max = *std::max_element(h.begin(), h.end());
  return decompose_device_impl(ctx, dX, m, n, ldx, &c, d_diag, dY, dT, h_selected, h_history,
                               result, nullptr, diag_max);
}

namespace {
// Device leading dimension of an uploaded X: columns stay 16-byte aligned.
long long upload_ld(long long m, bool f32) { return f32 ? (m + 3) / 4 * 4 : (m % 2 == 0 ? m : m + 1); }

// The host entry after the upload: X already sits in dXbuf (ld = upload_ld);
// runs the decompose and brings Y/T/selected/history back (Y and T stream out
// during the loop when the host buffers are page-locked).
int run_uploaded(rbd_ctx_t ctx, void* dXbuf, int64_t m, int64_t n, const rbd_config_t* cfg,
                 const double* h_diag, int64_t diag_len, double* hY, double* hT, int64_t* h_selected,
                 double* h_history, rbd_result_t* result, bool f32);

int decompose_host_impl(rbd_ctx_t ctx, const double* hX, int64_t m, int64_t n, int64_t ldx,
                        const rbd_config_t* cfg, const double* h_diag, int64_t diag_len,
                        double* hY, double* hT, int64_t* h_selected, double* h_history,
                        rbd_result_t* result, const float* hXf = nullptr) {
  if (!ctx || !cfg) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: null context/config");
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: matrix must be non-empty");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "decompose: ldx < m");
  CU(cudaSetDevice(ctx->device));
  const size_t es = hXf ? sizeof(float) : sizeof(double);
  const long long ldd = upload_ld(m, hXf != nullptr);
  TRY(ensure(ctx->hX, es * ldd * n));
  cudaError_t e = cudaMemcpy2DAsync(ctx->hX.p, es * ldd, hXf ? (const void*)hXf : (const void*)hX,
                                    es * ldx, es * m, n, cudaMemcpyHostToDevice, ctx->stream);
  if (e != cudaSuccess) return set_err(RBD_ERR_CUDA, std::string("H2D X: ") + cudaGetErrorString(e));
  return run_uploaded(ctx, ctx->hX.p, m, n, cfg, h_diag, diag_len, hY, hT, h_selected, h_history,
                      result, hXf != nullptr);
}

int run_uploaded(rbd_ctx_t ctx, void* dXbuf, int64_t m, int64_t n, const rbd_config_t* cfg,
                 const double* h_diag, int64_t diag_len, double* hY, double* hT, int64_t* h_selected,
                 double* h_history, rbd_result_t* result, bool f32) {
  const long long d_cap = std::max<long long>(1, std::min<long long>(cfg->d_max, n));
  const long long ldd = upload_ld(m, f32);
  const float* dXf = f32 ? reinterpret_cast<const float*>(dXbuf) : nullptr;   // fp32 storage mode
  TRY(ensure(ctx->hY, sizeof(double) * m * d_cap));
  TRY(ensure(ctx->hT, sizeof(double) * d_cap * n));
  double* dX = reinterpret_cast<double*>(dXbuf);
  double* dY = ptr<double>(ctx->hY);
  double* dT = ptr<double>(ctx->hT);
  cudaError_t e = cudaSuccess;
  rbd_result_t r{};
  int rc;
  bool t_streamed = false;
  if (h_diag || diag_len != 0) {
    TRY(check_diagonal(h_diag, diag_len));
    TRY(ensure(ctx->wd_diag, sizeof(double) * diag_len));
    CU(cudaMemcpyAsync(ctx->wd_diag.p, h_diag, sizeof(double) * diag_len, cudaMemcpyHostToDevice,
                       ctx->stream));
    rc = rbd_decompose_diag_device(ctx, dX, m, n, ldd, cfg, ptr<double>(ctx->wd_diag), diag_len,
                                   dY, dT, h_selected, h_history, &r);
  } else {
    ctx->ystream_dst = nullptr;
    ctx->tstream_dst = nullptr;
    if (hY) {   // page-locked Y: columns (and T rows) stream out while the loop runs
      cudaPointerAttributes pa{};
      if (cudaPointerGetAttributes(&pa, hY) == cudaSuccess && pa.type == cudaMemoryTypeHost) {
        ctx->ystream_dst = hY;
        if (hT && cudaPointerGetAttributes(&pa, hT) == cudaSuccess &&
            pa.type == cudaMemoryTypeHost)
          ctx->tstream_dst = hT;
        else
          cudaGetLastError();
      } else {
        cudaGetLastError();
      }
    }
    rc = dXf ? decompose_device_impl(ctx, nullptr, m, n, ldd, cfg, nullptr, dY, dT, h_selected,
                                     h_history, &r, dXf)
             : rbd_decompose_device(ctx, dX, m, n, ldd, cfg, dY, dT, h_selected, h_history, &r);
    t_streamed = ctx->tstream_dst != nullptr;
    ctx->ystream_dst = nullptr;
    ctx->tstream_dst = nullptr;
  }
  const long long y_done = (rc == RBD_OK) ? std::min<long long>(ctx->ystream_copied, r.d) : 0;
  const long long t_done = t_streamed ? y_done : 0;
  ctx->ystream_copied = 0;
  // dY was allocated with d_cap columns; the device call writes at most d_cap
  if (rc == RBD_OK) {
    if (hY && r.d > y_done)
      e = cudaMemcpyAsync(hY + y_done * m, dY + y_done * m, sizeof(double) * m * (r.d - y_done),
                          cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && y_done > 0 && ctx->copy_stream)
      e = cudaStreamSynchronize(ctx->copy_stream);   // the streamed columns
    if (e == cudaSuccess && hT && r.d > t_done)
      e = cudaMemcpyAsync(hT + t_done * n, dT + t_done * n, sizeof(double) * (r.d - t_done) * n,
                          cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = set_err(RBD_ERR_CUDA, std::string("D2H model: ") + cudaGetErrorString(e));
    if (result) *result = r;
  }
  return rc;
}

}  // namespace

int rbd_decompose_host(rbd_ctx_t ctx, const double* hX, int64_t m, int64_t n, int64_t ldx,
                       const rbd_config_t* cfg, double* hY, double* hT, int64_t* h_selected,
                       double* h_history, rbd_result_t* result) {
  return decompose_host_impl(ctx, hX, m, n, ldx, cfg, nullptr, 0, hY, hT, h_selected, h_history,
                             result);
}

int rbd_decompose_host_f32(rbd_ctx_t ctx, const float* hX, int64_t m, int64_t n, int64_t ldx,
                           const rbd_config_t* cfg, double* hY, double* hT, int64_t* h_selected,
                           double* h_history, rbd_result_t* result) {
  if (!hX) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: null X");
  return decompose_host_impl(ctx, nullptr, m, n, ldx, cfg, nullptr, 0, hY, hT, h_selected,
                             h_history, result, hX);
}

namespace {
// Pipelined host entry: the upload of matrix i+1 (second stream, copy engine)
// overlaps the greedy loop of matrix i; two device X buffers alternate. Each
// decompose is synchronous, so buffer (i+1) % 2 — last read by decompose
// i-1 — is free when its upload is enqueued.
int decompose_host_many_impl(rbd_ctx_t ctx, int64_t count, const void* const* hX, int64_t m,
                             int64_t n, int64_t ldx, const rbd_config_t* cfg, double* const* hY,
                             double* const* hT, int64_t* const* h_selected,
                             double* const* h_history, rbd_result_t* results, bool f32) {
  if (!ctx || !cfg) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: null context/config");
  if (count < 0 || (count > 0 && !hX)) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose_many: bad list");
  if (count == 0) return RBD_OK;
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: matrix must be non-empty");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "decompose: ldx < m");
  for (int64_t i = 0; i < count; ++i)
    if (!hX[i]) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: null X");
  CU(cudaSetDevice(ctx->device));
  const size_t es = f32 ? sizeof(float) : sizeof(double);
  const long long ldd = upload_ld(m, f32);
  const size_t bytes = es * (size_t)ldd * (size_t)n;
  TRY(ensure(ctx->hX2, 2 * bytes));
  if (!ctx->up_stream) CU(cudaStreamCreateWithFlags(&ctx->up_stream, cudaStreamNonBlocking));
  cudaEvent_t up[2];
  CU(cudaEventCreateWithFlags(&up[0], cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&up[1], cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t* e;
    cudaStream_t s;
    ~EvGuard() {
      cudaStreamSynchronize(s);   // no upload may outlive the call
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } guard{up, ctx->up_stream};
  char* buf = static_cast<char*>(ctx->hX2.p);
  auto upload = [&](int64_t i) -> int {
    cudaError_t e = cudaMemcpy2DAsync(buf + (i % 2) * bytes, es * ldd, hX[i], es * ldx, es * m, n,
                                      cudaMemcpyHostToDevice, ctx->up_stream);
    if (e == cudaSuccess) e = cudaEventRecord(up[i % 2], ctx->up_stream);
    if (e != cudaSuccess) return set_err(RBD_ERR_CUDA, std::string("H2D X: ") + cudaGetErrorString(e));
    return RBD_OK;
  };
  TRY(upload(0));
  for (int64_t i = 0; i < count; ++i) {
    CU(cudaStreamWaitEvent(ctx->stream, up[i % 2], 0));
    if (i + 1 < count) TRY(upload(i + 1));
    TRY(run_uploaded(ctx, buf + (i % 2) * bytes, m, n, cfg, nullptr, 0, hY ? hY[i] : nullptr,
                     hT ? hT[i] : nullptr, h_selected ? h_selected[i] : nullptr,
                     h_history ? h_history[i] : nullptr, results ? &results[i] : nullptr, f32));
  }
  return RBD_OK;
}
}  // namespace

int rbd_decompose_host_many(rbd_ctx_t ctx, int64_t count, const double* const* hX, int64_t m,
                            int64_t n, int64_t ldx, const rbd_config_t* cfg, double* const* hY,
                            double* const* hT, int64_t* const* h_selected, double* const* h_history,
                            rbd_result_t* results) {
  return decompose_host_many_impl(ctx, count, reinterpret_cast<const void* const*>(hX), m, n, ldx,
                                  cfg, hY, hT, h_selected, h_history, results, false);
}

int rbd_decompose_host_many_f32(rbd_ctx_t ctx, int64_t count, const float* const* hX, int64_t m,
                                int64_t n, int64_t ldx, const rbd_config_t* cfg, double* const* hY,
                                double* const* hT, int64_t* const* h_selected,
                                double* const* h_history, rbd_result_t* results) {
  return decompose_host_many_impl(ctx, count, reinterpret_cast<const void* const*>(hX), m, n, ldx,
                                  cfg, hY, hT, h_selected, h_history, results, true);
}

int rbd_decompose_diag_host(rbd_ctx_t ctx, const double* hX, int64_t m, int64_t n, int64_t ldx,
                            const rbd_config_t* cfg, const double* h_diag, int64_t diag_len,
                            double* hY, double* hT, int64_t* h_selected, double* h_history,
                            rbd_result_t* result) {
  if (!h_diag && diag_len > 0) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: null diagonal");
  if (diag_len <= 0) return set_err(RBD_ERR_INVALID_ARGUMENT, "diagonal weight must be non-empty");
  return decompose_host_impl(ctx, hX, m, n, ldx, cfg, h_diag, diag_len, hY, hT, h_selected,
                             h_history, result);
}

int rbd_mgs_project(rbd_ctx_t ctx, const double* dv, int64_t m, const double* dB, int64_t k,
                    int64_t ldb, double breakdown_tol, int reorthogonalize, double* dxi,
                    double* norm, int* ok) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1) return set_err(RBD_ERR_DIMENSION_MISMATCH, "mgs_project: vector length != basis row count");
  if (k > 0 && ldb < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "mgs_project: ldb < m");
  CU(cudaSetDevice(ctx->device));
  // the extension kernels read the basis with ld m; repack when ldb != m
  const double* B = dB;
  DevBuf packed;
  const long long S = cdiv(m, kChunk);
  TRY(ensure(ctx->scratch1, sizeof(DevState) + sizeof(double) * (3 * (k + 1) + m + gemv_grid(m) +
                                                                  S * std::max<long long>(k, 1))));
  if (k > 0 && ldb != m) {
    TRY(ensure(packed, sizeof(double) * m * k));
    CU(cudaMemcpy2DAsync(packed.p, sizeof(double) * m, dB, sizeof(double) * ldb, sizeof(double) * m,
                         k, cudaMemcpyDeviceToDevice, ctx->stream));
    B = ptr<double>(packed);
  }
  char* base = static_cast<char*>(ctx->scratch1.p);
  DevState* st = reinterpret_cast<DevState*>(base);
  double* c = reinterpret_cast<double*>(base + sizeof(DevState));
  double* p = c + (k + 1);
  double* w = p + (k + 1);
  double* nrm = w + m;
  double* partial = nrm + gemv_grid(m);
  DevState hs{};
  hs.d = k;
  hs.d_max = k + 1;
  hs.breakdown_tol = breakdown_tol;
  hs.cfg_reorth = reorthogonalize ? 1 : 0;
  *ctx->h_state = hs;
  CU(cudaMemcpyAsync(st, ctx->h_state, sizeof(DevState), cudaMemcpyHostToDevice, ctx->stream));
  k_norm2_single<<<1, kThreads, 0, ctx->stream>>>(dv, m, st);
  ctx->launches++;
  if (k > 0) {
    const int vec = (m % 2 == 0 && aligned16(B) && aligned16(dv)) ? 2 : 1;
    SweepArgs s{};
    s.A = B;
    s.lda = m;
    s.m = m;
    s.ncols = k;
    s.v = dv;
    s.partial = partial;
    s.pstride = k;
    s.st = st;
    s.gate = GATE_NONE;
    TRY(launch_sweep(ctx, s, vec, MODE_DOT, false, k));
    k_coef_combine<<<(unsigned)cdiv(k, 256), 256, 0, ctx->stream>>>(partial, S, k, c, st, GATE_NONE);
    ctx->launches++;
  }
  ExtBufs b{};
  b.B = B;
  b.m = m;
  b.dcap = std::max<long long>(k, 1);
  b.X = nullptr;
  b.v = dv;
  b.c = c;
  b.w = w;
  b.p = p;
  b.nrm = nrm;
  b.partial = partial;
  b.ybase = dxi;
  b.use_d = 0;
  b.selected = nullptr;
  b.st = st;
  TRY(enqueue_extension(ctx, b));
  CU(cudaMemcpyAsync(ctx->h_state, st, sizeof(DevState), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  release(packed);
  hs = *ctx->h_state;
  if (ok) *ok = hs.breakdown ? 0 : 1;
  if (norm) *norm = hs.wnorm;
  return RBD_OK;
}

}  // extern "C"

extern "C" {

int rbd_mgs_project_host(rbd_ctx_t ctx, const double* hv, int64_t m, const double* hB, int64_t k,
                         int64_t ldb, double breakdown_tol, int reorthogonalize, double* hxi,
                         double* norm, int* ok) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1) return set_err(RBD_ERR_DIMENSION_MISMATCH, "mgs_project: vector length != basis row count");
  if (k > 0 && ldb < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "mgs_project: vector length != basis row count");
  CU(cudaSetDevice(ctx->device));
  DevBuf &bv = ctx->hs[0], &bB = ctx->hs[1], &bx = ctx->hs[2];   // kept between calls
  auto fin = [&](int rc) { return rc; };
  int rc;
  if ((rc = ensure(bv, sizeof(double) * m)) || (rc = ensure(bx, sizeof(double) * m)) ||
      (rc = ensure(bB, sizeof(double) * m * std::max<int64_t>(k, 1))))
    return fin(rc);
  if (cudaMemcpyAsync(bv.p, hv, sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream) ||
      (k > 0 && cudaMemcpy2DAsync(bB.p, sizeof(double) * m, hB, sizeof(double) * ldb,
                                  sizeof(double) * m, k, cudaMemcpyHostToDevice, ctx->stream)))
    return fin(set_err(RBD_ERR_CUDA, "mgs_project_host: H2D failed"));
  int okv = 0;
  double nv = 0.0;
  rc = rbd_mgs_project(ctx, ptr<double>(bv), m, ptr<double>(bB), k, m, breakdown_tol,
                       reorthogonalize, ptr<double>(bx), &nv, &okv);
  if (rc) return fin(rc);
  if (okv && hxi && cudaMemcpy(hxi, bx.p, sizeof(double) * m, cudaMemcpyDeviceToHost))
    return fin(set_err(RBD_ERR_CUDA, "mgs_project_host: D2H failed"));
  if (ok) *ok = okv;
  if (norm) *norm = nv;
  return fin(RBD_OK);
}

}  // extern "C"
