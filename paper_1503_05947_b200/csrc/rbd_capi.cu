// rbd_capi.cu — host runtime of the B200 RBD path behind the C ABI in
// include/rbd_cuda.h: context, scratch management, the CUDA-graph-captured
// greedy step loop, the workspace API and out-of-sample projection.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "rbd_cuda.h"
#include "rbd_internal.h"
#include "rbd_device.cuh"
#include "rbd_project.cuh"
#include "rbd_persistent.cuh"
#include "rbd_project_tc.cuh"
#include "rbd_weighted.cuh"
#include "rbd_classify.cuh"
#include "rbd_compress_dmma.cuh"

#include <cudaTypedefs.h>

using namespace rbdk;

void rbd_comm_release(rbd_ctx_t ctx);

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return set_err(e_ == cudaErrorMemoryAllocation ? RBD_ERR_OUT_OF_MEMORY : RBD_ERR_CUDA, \
                     std::string(#call) + ": " + cudaGetErrorString(e_));                 \
  } while (0)

#define TRY(expr)            \
  do {                       \
    int s_ = (expr);         \
    if (s_ != RBD_OK) return s_; \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

int ensure(DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.bytes >= bytes) return RBD_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e != cudaSuccess)
    return set_err(RBD_ERR_OUT_OF_MEMORY, std::string("cudaMalloc(") + std::to_string(bytes) +
                                              "): " + cudaGetErrorString(e));
  b.bytes = bytes;
  return RBD_OK;
}

void release(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}

template <typename T>
T* ptr(DevBuf& b) {
  return static_cast<T*>(b.p);
}

long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct GraphKey {
  const void* X = nullptr;
  const void* Y = nullptr;
  const void* T = nullptr;
  long long m = 0, n = 0, ldx = 0, d_max = 0;
  const void* bufs[8] = {};
  cudaStream_t stream = nullptr;
  int steps = 0;
  bool operator==(const GraphKey& o) const {
    if (X != o.X || Y != o.Y || T != o.T || m != o.m || n != o.n || ldx != o.ldx ||
        d_max != o.d_max || stream != o.stream || steps != o.steps)
      return false;
    for (int i = 0; i < 8; ++i)
      if (bufs[i] != o.bufs[i]) return false;
    return true;
  }
};

}  // namespace

struct rbd_ctx_s {
  int device = 0;
  int nsm = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  DevBuf partial, rec, counter, state, colsq, resid, w, c, p, nrm, hist, sel, out_rec, scratch1;
  DevBuf hX, hY, hT;  // cached device copies for the host entry
  DevBuf ppart;       // fused-extension partials
  DevState* h_state = nullptr;  // pinned
  // host entry with a page-locked Y: the loop posts its progress to a mapped
  // word and finished Y columns are copied out on a second stream meanwhile
  long long* h_progress = nullptr;
  long long* d_progress = nullptr;
  cudaStream_t copy_stream = nullptr;
  double* ystream_dst = nullptr;   // host Y (ld m) to stream into, or null
  double* tstream_dst = nullptr;   // host T (row-major, n per row), or null
  long long ystream_copied = 0;    // Y columns / T rows already copied (or in flight)
  Rec* h_rec = nullptr;         // pinned
  cudaGraphExec_t gexec = nullptr;
  GraphKey gkey;
  long long graph_nodes = 0;
  long long launches = 0;
  int occ_sweep2 = 2, occ_sweep1 = 2;
  int fused_grid_cap = 296;
  int persist_occ2 = 0, persist_occ1 = 0;  // co-resident CTAs/SM of the persistent kernel
  int path = 0;                            // 0 persistent, 1 graph of per-phase kernels
  DevBuf bar;                              // grid-barrier words
  DevBuf ctl, gcnt, ygcnt;                 // persistent loop: ctl words, p (x2), CTA records
  DevBuf rdy;                              // persistent loop: P1 readiness counters
  // diagonal-weight loop (rbd_weighted.cuh): a o xi, xi'A xi partials, YAX row
  // partials, YAY row, YAX (d_max x n), cross, quad, col_sq_A, host-entry diag
  DevBuf wd_axi, wd_yy, wd_part2, wd_yrow, wd_yax, wd_cross, wd_quad, wd_colsq, wd_diag;
  DevBuf wd_ppart2, wd_q, wd_yay;           // persistent weighted loop: Y'(a o w1), YAY
  DevBuf forced;                             // rbd_set_forced_selection (test instrumentation)
  std::vector<long long> forced_h;
  DevBuf nn_part, nn_coords;               // classify: split minima, query coordinates
  DevBuf pj_ws;                            // K5 split-K partial slices
  DevBuf send, recv;                       // sharded mode: payload exchange buffers
  // multi-GPU
  void* comm = nullptr;                    // ncclComm_t (dlopen'ed NCCL)
  int rank = 0, world = 1;
  std::vector<rbd_ctx_s*> virt;            // virtual ranks (single-device sharded mode)
};

struct rbd_ws_s {
  rbd_ctx_t ctx;
  const double* X;
  long long m, n, ldx, cap, d;
  DevBuf T, colsq, resid, partial, rec, counter, out, tmp;
  DevBuf Xown;   // host-entry workspaces own a device copy of X
  // diagonal weight (kind 1, workspace.hpp:18-30): the weight, the basis vectors
  // passed to extend (for Y'AY), a o xi scratch and its partials, Y'AY (cap x cap),
  // a row scratch
  int kind = 0;
  DevBuf diag, basis, axi, yy, yay, row;
};

namespace {

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
size_t persist_smem(long long dcap, bool diag = false) {
  const size_t d = (size_t)std::max<long long>(dcap, 1);
  return sizeof(double) * (2 * (d + 16 * kWarps) + (diag ? 2 * (d + 1) : 0));
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

int persistent_grid(rbd_ctx_t ctx, int vec, long long d_max, bool diag = false) {
  int occ = 0;
  const size_t smem = persist_smem(d_max, diag);
  if (diag)
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
  const int vec = (L.ldx % 2 == 0 && L.m % 2 == 0 && aligned16(L.X) && aligned16(L.Y) &&
                   aligned16(ctx->w.p) && (!diag || aligned16(ctx->wd_axi.p))) ? 2 : 1;
  const int grid = persistent_grid(ctx, vec, L.d_max, diag != nullptr);
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
  if (getenv("RBD_PHASE_TIMING")) {
    TRY(ensure(ctx->scratch1, 256));
    cudaMemsetAsync(ctx->scratch1.p, 0, 128, ctx->stream);
    a.phase_ns = ptr<unsigned long long>(ctx->scratch1);
  }
  a.trace = nullptr;
  DevBuf tracebuf;
  if (const char* ts = getenv("RBD_TRACE_STEP")) {
    TRY(ensure(tracebuf, sizeof(unsigned long long) * (size_t)grid * kTraceWords));
    cudaMemsetAsync(tracebuf.p, 0, sizeof(unsigned long long) * (size_t)grid * kTraceWords, ctx->stream);
    a.trace = ptr<unsigned long long>(tracebuf);
    a.trace_step = atoll(ts);
  }
  void* args[] = {&a};
  const size_t smem = persist_smem(L.d_max, diag != nullptr);
  void* fn = diag ? (vec == 2 ? (void*)k_rbd_persistent<2, false, true>
                              : (void*)k_rbd_persistent<1, false, true>)
                  : (vec == 2 ? (void*)k_rbd_persistent<2, false> : (void*)k_rbd_persistent<1, false>);
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
                        bool diag_supplied = false) {
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

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* rbd_last_error(void) { return g_err.c_str(); }

// for the library's other translation units (csrc/rbd_internal.h)
__attribute__((visibility("hidden"))) int rbd_internal_set_error(int code, const char* msg) {
  return set_err(code, msg);
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
  cudaFuncSetAttribute(k_rbd_persistent<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)fused_smem(kFMaxCoef));
  cudaFuncSetAttribute(k_rbd_persistent<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)fused_smem(kFMaxCoef));
  cudaFuncSetAttribute(k_rbd_persistent<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)fused_smem(kFMaxCoef));
  cudaFuncSetAttribute(k_rbd_persistent<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)fused_smem(kFMaxCoef));
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
                  &ctx->hX,      &ctx->hY,   &ctx->hT,      &ctx->ppart, &ctx->bar,
                  &ctx->wd_axi,  &ctx->wd_yy, &ctx->wd_part2, &ctx->wd_yrow, &ctx->wd_yax,
                  &ctx->wd_cross, &ctx->wd_quad, &ctx->wd_colsq, &ctx->wd_diag,
                  &ctx->wd_ppart2, &ctx->wd_q, &ctx->wd_yay, &ctx->forced,
                  &ctx->nn_part, &ctx->nn_coords, &ctx->pj_ws,
                  &ctx->ctl,     &ctx->gcnt, &ctx->ygcnt,   &ctx->rdy,   &ctx->send,  &ctx->recv};
  for (DevBuf* b : bl) release(*b);
  if (ctx->h_state) cudaFreeHost(ctx->h_state);
  if (ctx->h_progress) cudaFreeHost(ctx->h_progress);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
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
                          int64_t* h_selected, double* h_history, rbd_result_t* result) {
  if (!ctx || !cfg) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: null context/config");
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: matrix must be non-empty");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "decompose: ldx < m");
  CU(cudaSetDevice(ctx->device));
  const long long d_cap = std::max<long long>(1, std::min<long long>(cfg->d_max, n));
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
  CU(cudaMemsetAsync(st, 0, sizeof(DevState), ctx->stream));
  CU(cudaEventRecord(ev0, ctx->stream));
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
  DevState hs = *ctx->h_state;
  double init_ms = 0.0;
  {
    float t = 0.f;
    cudaEventElapsedTime(&t, ev0, ev1);
    init_ms = t;
  }
  TRY(validate_after_init(cfg, m, n, hs, diag != nullptr));
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

  LoopBufs L{dX, m, n, ldx, cfg->d_max, dY, dT};
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
int check_diagonal(const double* h, int64_t len) {
  if (len <= 0) return set_err(RBD_ERR_INVALID_ARGUMENT, "diagonal weight must be non-empty");
  for (int64_t i = 0; i < len; ++i)
    if (!(h[i] > 0.0) || !std::isfinite(h[i]))
      return set_err(RBD_ERR_INVALID_ARGUMENT,
                     "diagonal weight entries must be strictly positive and finite");
  return RBD_OK;
}
}  // namespace

int rbd_decompose_device(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx,
                         const rbd_config_t* cfg, double* dY, double* dT, int64_t* h_selected,
                         double* h_history, rbd_result_t* result) {
  return decompose_device_impl(ctx, dX, m, n, ldx, cfg, nullptr, dY, dT, h_selected, h_history,
                               result);
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
  return decompose_device_impl(ctx, dX, m, n, ldx, &c, d_diag, dY, dT, h_selected, h_history,
                               result);
}

namespace {
int decompose_host_impl(rbd_ctx_t ctx, const double* hX, int64_t m, int64_t n, int64_t ldx,
                        const rbd_config_t* cfg, const double* h_diag, int64_t diag_len,
                        double* hY, double* hT, int64_t* h_selected, double* h_history,
                        rbd_result_t* result) {
  if (!ctx || !cfg) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: null context/config");
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: matrix must be non-empty");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "decompose: ldx < m");
  CU(cudaSetDevice(ctx->device));
  const long long d_cap = std::max<long long>(1, std::min<long long>(cfg->d_max, n));
  const long long ldd = (m % 2 == 0) ? m : m + 1;  // keep columns 16-byte aligned on device
  TRY(ensure(ctx->hX, sizeof(double) * ldd * n));
  TRY(ensure(ctx->hY, sizeof(double) * m * d_cap));
  TRY(ensure(ctx->hT, sizeof(double) * d_cap * n));
  double* dX = ptr<double>(ctx->hX);
  double* dY = ptr<double>(ctx->hY);
  double* dT = ptr<double>(ctx->hT);
  cudaError_t e = cudaMemcpy2DAsync(dX, sizeof(double) * ldd, hX, sizeof(double) * ldx,
                                    sizeof(double) * m, n, cudaMemcpyHostToDevice, ctx->stream);
  if (e != cudaSuccess) return set_err(RBD_ERR_CUDA, std::string("H2D X: ") + cudaGetErrorString(e));
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
    rc = rbd_decompose_device(ctx, dX, m, n, ldd, cfg, dY, dT, h_selected, h_history, &r);
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

// ---------------------------------------------------------------------------
// Workspace API
// ---------------------------------------------------------------------------
int rbd_ws_init(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx, int64_t cap,
                rbd_ws_t* out) {
  if (!ctx || !out) return set_err(RBD_ERR_INVALID_ARGUMENT, "null argument");
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "workspace_init: empty matrix");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "workspace_init: ldx < m");
  CU(cudaSetDevice(ctx->device));
  auto* ws = new rbd_ws_s();
  ws->ctx = ctx;
  ws->X = dX;
  ws->m = m;
  ws->n = n;
  ws->ldx = ldx;
  ws->cap = std::max<int64_t>(cap, 1);
  ws->d = 0;
  const long long S = cdiv(m, kChunk);
  int rc = RBD_OK;
  if ((rc = ensure(ws->T, sizeof(double) * ws->cap * n)) ||
      (rc = ensure(ws->colsq, sizeof(double) * n)) || (rc = ensure(ws->resid, sizeof(double) * n)) ||
      (rc = ensure(ws->partial, sizeof(double) * S * n)) ||
      (rc = ensure(ws->rec, sizeof(Rec) * (size_t)ctx->nsm * 8)) ||
      (rc = ensure(ws->counter, 64)) || (rc = ensure(ws->out, 64)) ||
      (rc = ensure(ws->tmp, sizeof(DevState) + 64))) {
    rbd_ws_destroy(ws);
    return rc;
  }
  cudaMemsetAsync(ws->counter.p, 0, 64, ctx->stream);
  cudaMemsetAsync(ws->tmp.p, 0, sizeof(DevState), ctx->stream);
  rc = enqueue_init(ctx, dX, m, n, ldx, ptr<double>(ws->partial), ptr<double>(ws->colsq),
                    ptr<double>(ws->resid), ptr<DevState>(ws->tmp));
  if (rc == RBD_OK && cudaStreamSynchronize(ctx->stream) != cudaSuccess)
    rc = set_err(RBD_ERR_CUDA, "workspace_init: kernel failure");
  if (rc != RBD_OK) {
    rbd_ws_destroy(ws);
    return rc;
  }
  *out = ws;
  return RBD_OK;
}

int rbd_ws_destroy(rbd_ws_t ws) {
  if (!ws) return RBD_OK;
  DevBuf* bl[] = {&ws->T,       &ws->colsq, &ws->resid, &ws->partial, &ws->rec,
                  &ws->counter, &ws->out,   &ws->tmp,   &ws->Xown,    &ws->diag,
                  &ws->basis,   &ws->axi,   &ws->yy,    &ws->yay,     &ws->row};
  for (DevBuf* b : bl) release(*b);
  delete ws;
  return RBD_OK;
}

int64_t rbd_ws_d(rbd_ws_t ws) { return ws ? ws->d : 0; }

int rbd_ws_extend(rbd_ws_t ws, const double* dxi) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  if (ws->d >= ws->cap) return set_err(RBD_ERR_INVALID_ARGUMENT, "workspace_extend: capacity exhausted");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  if (ws->kind == 1) {   // diagonal, workspace.cpp:61-79
    const long long m = ws->m, n = ws->n, d = ws->d, S = cdiv(m, kChunk);
    double* basis = ptr<double>(ws->basis);
    CU(cudaMemcpyAsync(basis + d * m, dxi, sizeof(double) * m, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    // a o xi (weight.cpp:83) and xi'A xi (:75): k_diag_vec reads column st->d of
    // its "Y" argument; the workspace's scratch state has d = 0, done = 0
    DevState* st0 = ptr<DevState>(ws->tmp);
    const int gv = diag_vec_grid(ctx, m);
    k_diag_vec<<<gv, kThreads, 0, ctx->stream>>>(basis + d * m, m, ptr<double>(ws->diag),
                                                 ptr<double>(ws->axi), ptr<double>(ws->yy), st0);
    ctx->launches++;
    // YAX row d = X'(a o xi) (:66)
    const int vx = (ws->ldx % 2 == 0 && aligned16(ws->X) && aligned16(ws->axi.p)) ? 2 : 1;
    SweepArgs s{};
    s.A = ws->X;
    s.lda = ws->ldx;
    s.m = m;
    s.ncols = n;
    s.v = ptr<double>(ws->axi);
    s.partial = ptr<double>(ws->partial);
    s.pstride = n;
    s.gate = GATE_NONE;
    TRY(launch_sweep(ctx, s, vx, MODE_DOT, true, n));
    const int gr = (int)std::max<long long>(1, std::min<long long>(cdiv(n, 256), (long long)ctx->nsm * 4));
    k_rowsum<<<gr, 256, 0, ctx->stream>>>(ptr<double>(ws->partial), S, n, ptr<double>(ws->T) + d * n);
    ctx->launches++;
    // YAY row d (:69-75): the earlier basis vectors against a o xi
    if (d > 0) {
      const int vb = (m % 2 == 0 && aligned16(ws->basis.p) && aligned16(ws->axi.p)) ? 2 : 1;
      SweepArgs b{};
      b.A = basis;
      b.lda = m;
      b.m = m;
      b.ncols = d;
      b.v = ptr<double>(ws->axi);
      b.partial = ptr<double>(ws->partial);
      b.pstride = d;
      b.gate = GATE_NONE;
      TRY(launch_sweep(ctx, b, vb, MODE_DOT, false, d));
      k_rowsum<<<(unsigned)std::max<long long>(1, cdiv(d, 256)), 256, 0, ctx->stream>>>(
          ptr<double>(ws->partial), S, d, ptr<double>(ws->row));
      ctx->launches++;
    }
    k_yay_row<<<(unsigned)std::max<long long>(1, cdiv(d, 256)), 256, 0, ctx->stream>>>(
        ptr<double>(ws->row), d, ptr<double>(ws->yy), gv, ptr<double>(ws->yay), ws->cap);
    ctx->launches++;
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(ctx->stream));
    ws->d += 1;
    return RBD_OK;
  }
  const int vec = (ws->ldx % 2 == 0 && aligned16(ws->X) && aligned16(dxi)) ? 2 : 1;
  SweepArgs s{};
  s.A = ws->X;
  s.lda = ws->ldx;
  s.m = ws->m;
  s.ncols = ws->n;
  s.v = dxi;
  s.partial = ptr<double>(ws->partial);
  s.pstride = ws->n;
  s.st = nullptr;
  s.gate = GATE_NONE;
  TRY(launch_sweep(ctx, s, vec, MODE_DOT, true, ws->n));
  FinalizeArgs f{};
  f.partial = ptr<double>(ws->partial);
  f.S = cdiv(ws->m, kChunk);
  f.n = ws->n;
  f.T = ptr<double>(ws->T);
  f.krow = ws->d;
  f.r = ptr<double>(ws->resid);
  f.col_sq = ptr<double>(ws->colsq);
  f.st = nullptr;
  f.mode = 1;
  k_finalize<<<finalize_grid(ctx, ws->n), kThreads, 0, ctx->stream>>>(f);
  ctx->launches++;
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(ctx->stream));
  ws->d += 1;
  return RBD_OK;
}

int rbd_ws_scan(rbd_ws_t ws, double* e_cur, int64_t* argmax) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  const int g = finalize_grid(ctx, ws->n);
  k_scan_only<<<g, kThreads, 0, ctx->stream>>>(ptr<double>(ws->resid), ws->n, ptr<Rec>(ws->rec),
                                                ptr<unsigned>(ws->counter), ptr<Rec>(ws->out));
  ctx->launches++;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(ctx->h_rec, ws->out.p, sizeof(Rec), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (e_cur) *e_cur = ctx->h_rec->v;
  if (argmax) *argmax = ctx->h_rec->j;
  return RBD_OK;
}

int rbd_ws_error_sq(rbd_ws_t ws, int64_t j, const double* h_c, int64_t clen, double* out) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  if (j < 0 || j >= ws->n) return set_err(RBD_ERR_INDEX_OUT_OF_RANGE, "error_sq: column index out of range");
  if (clen != ws->d) return set_err(RBD_ERR_DIMENSION_MISMATCH, "error_sq: coefficient length != d");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  double* dc = reinterpret_cast<double*>(static_cast<char*>(ws->tmp.p) + sizeof(DevState));
  DevBuf cbuf;
  if (clen > 0) {
    TRY(ensure(cbuf, sizeof(double) * clen));
    CU(cudaMemcpyAsync(cbuf.p, h_c, sizeof(double) * clen, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (ws->kind == 1)
    k_error_sq_w<<<1, kThreads, 0, ctx->stream>>>(ptr<double>(ws->T), ws->n, ws->d, j,
                                                  ptr<double>(cbuf), ptr<double>(ws->yay), ws->cap,
                                                  ptr<double>(ws->colsq), dc);
  else
    k_error_sq<<<1, kThreads, 0, ctx->stream>>>(ptr<double>(ws->T), ws->n, ws->d, j,
                                                ptr<double>(cbuf), ptr<double>(ws->colsq), dc);
  ctx->launches++;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(out, dc, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  release(cbuf);
  return RBD_OK;
}

int rbd_ws_read(rbd_ws_t ws, double* h_col_sq, double* h_residual_sq, double* h_yax) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  if (h_col_sq) CU(cudaMemcpyAsync(h_col_sq, ws->colsq.p, sizeof(double) * ws->n, cudaMemcpyDeviceToHost, ctx->stream));
  if (h_residual_sq)
    CU(cudaMemcpyAsync(h_residual_sq, ws->resid.p, sizeof(double) * ws->n, cudaMemcpyDeviceToHost, ctx->stream));
  if (h_yax && ws->d > 0)
    CU(cudaMemcpyAsync(h_yax, ws->T.p, sizeof(double) * ws->d * ws->n, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return RBD_OK;
}

int rbd_ws_init_diag(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx,
                     int64_t cap, const double* d_diag, int64_t diag_len, rbd_ws_t* out) {
  if (!ctx || !out) return set_err(RBD_ERR_INVALID_ARGUMENT, "null argument");
  CU(cudaSetDevice(ctx->device));
  std::vector<double> h((size_t)std::max<int64_t>(diag_len, 0));
  if (diag_len > 0) {
    if (!d_diag) return set_err(RBD_ERR_INVALID_ARGUMENT, "workspace_init: null diagonal");
    CU(cudaMemcpyAsync(h.data(), d_diag, sizeof(double) * diag_len, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  TRY(check_diagonal(h.data(), diag_len));                              // weight.cpp:11-17
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "workspace_init: empty matrix");
  if (diag_len != m)                                                    // workspace.cpp:12-13
    return set_err(RBD_ERR_INCOMPATIBLE_WEIGHT, "weight dimension does not match matrix rows");
  rbd_ws_t ws = nullptr;
  TRY(rbd_ws_init(ctx, dX, m, n, ldx, cap, &ws));
  int rc = RBD_OK;
  const long long c = ws->cap;
  if ((rc = ensure(ws->diag, sizeof(double) * m)) || (rc = ensure(ws->basis, sizeof(double) * m * c)) ||
      (rc = ensure(ws->axi, sizeof(double) * m)) ||
      (rc = ensure(ws->yy, sizeof(double) * diag_vec_grid(ctx, m))) ||
      (rc = ensure(ws->yay, sizeof(double) * c * c)) ||
      (rc = ensure(ws->row, sizeof(double) * std::max<long long>(c, 1))) ||
      (rc = ensure(ws->partial, sizeof(double) * cdiv(m, kChunk) * std::max<long long>(n, c)))) {
    rbd_ws_destroy(ws);
    return rc;
  }
  ws->kind = 1;
  cudaMemcpyAsync(ws->diag.p, d_diag, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream);
  cudaMemsetAsync(ws->yay.p, 0, sizeof(double) * c * c, ctx->stream);
  // col_sq = diag(X'AX) (workspace.cpp:24-29), residual_sq = col_sq (:38)
  const int g = (int)std::max<long long>(1, std::min<long long>(n, (long long)ctx->nsm * 8));
  k_colsq_diag<<<g, kThreads, 0, ctx->stream>>>(dX, ldx, m, n, ptr<double>(ws->diag),
                                                ptr<double>(ws->colsq));
  ctx->launches++;
  cudaMemcpyAsync(ws->resid.p, ws->colsq.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream);
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    rbd_ws_destroy(ws);
    return set_err(RBD_ERR_CUDA, "workspace_init: kernel failure");
  }
  *out = ws;
  return RBD_OK;
}

int rbd_ws_scan_T(rbd_ws_t ws, const double* dT, double* e_cur, int64_t* argmax) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  if (ws->d > 0 && !dT) return set_err(RBD_ERR_DIMENSION_MISMATCH, "residual_scan: T shape does not match workspace");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  const int g = finalize_grid(ctx, ws->n);
  k_scan_T<<<g, kThreads, 0, ctx->stream>>>(ptr<double>(ws->T), dT, ws->n, ws->d,
                                            ws->kind == 1 ? ptr<double>(ws->yay) : nullptr, ws->cap,
                                            ptr<double>(ws->colsq), ptr<Rec>(ws->rec),
                                            ptr<unsigned>(ws->counter), ptr<Rec>(ws->out));
  ctx->launches++;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(ctx->h_rec, ws->out.p, sizeof(Rec), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (e_cur) *e_cur = ctx->h_rec->v;
  if (argmax) *argmax = ctx->h_rec->j;
  return RBD_OK;
}

int rbd_ws_scan_T_host(rbd_ws_t ws, const double* hT, double* e_cur, int64_t* argmax) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  DevBuf tb;
  if (ws->d > 0) {
    TRY(ensure(tb, sizeof(double) * ws->d * ws->n));
    if (cudaMemcpyAsync(tb.p, hT, sizeof(double) * ws->d * ws->n, cudaMemcpyHostToDevice,
                        ctx->stream) != cudaSuccess) {
      release(tb);
      return set_err(RBD_ERR_CUDA, "residual_scan: H2D failed");
    }
  }
  const int rc = rbd_ws_scan_T(ws, ws->d > 0 ? ptr<double>(tb) : nullptr, e_cur, argmax);
  release(tb);
  return rc;
}

int rbd_ws_read_yay(rbd_ws_t ws, double* h_yay) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  if (ws->kind != 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "read_yay: identity workspace (Y'AY = I)");
  rbd_ctx_t ctx = ws->ctx;
  CU(cudaSetDevice(ctx->device));
  if (ws->d > 0)
    CU(cudaMemcpy2DAsync(h_yay, sizeof(double) * ws->d, ws->yay.p, sizeof(double) * ws->cap,
                         sizeof(double) * ws->d, ws->d, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return RBD_OK;
}

// ---------------------------------------------------------------------------
// Out-of-sample compression (K5) and reconstruct
// ---------------------------------------------------------------------------
int rbd_project_batch(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                      const double* dXn, int64_t N, int64_t ldx, double* dTn, double* d_err) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || N < 0) return set_err(RBD_ERR_DIMENSION_MISMATCH, "project: bad sizes");
  if (ldy < m || ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "project: vector length != m");
  if (N == 0) return RBD_OK;
  CU(cudaSetDevice(ctx->device));
  long long nl = 0;
  if (d_err) TRY(ensure(ctx->scratch1, sizeof(double) * (size_t)std::max<int64_t>(N, 32)));
  // split the K = m reduction when the DMMA grid would leave a partial last wave
  int sk = rbdk::project_splitk(m, d, N, ctx->nsm);
  if (sk > 1 && ensure(ctx->pj_ws, sizeof(double) * (size_t)(sk - 1) * (size_t)(d * N + N)) != RBD_OK)
    sk = 1;
  int rc = rbdk::launch_project_f64(dY, m, d, ldy, dXn, N, ldx, dTn, d_err, ctx->stream, &nl,
                                    d_err ? ptr<double>(ctx->scratch1) : nullptr, sk,
                                    sk > 1 ? ptr<double>(ctx->pj_ws) : nullptr);
  ctx->launches += nl;
  if (rc != 0) return set_err(RBD_ERR_CUDA, std::string("project kernel: ") + cudaGetErrorString((cudaError_t)rc));
  return RBD_OK;
}

int rbd_nearest_columns(rbd_ctx_t ctx, const double* dC, int64_t d, int64_t Q, int64_t ldc,
                        const double* dT, int64_t n_train, int64_t* d_best, double* d_dist) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (d < 1 || n_train < 1 || Q < 0 || ldc < d)
    return set_err(RBD_ERR_DIMENSION_MISMATCH, "nearest: bad sizes");
  if (Q == 0) return RBD_OK;
  if (!dC || !dT || !d_best) return set_err(RBD_ERR_INVALID_ARGUMENT, "nearest: null buffer");
  CU(cudaSetDevice(ctx->device));
  const long long gx = cdiv(Q, kNnTile);
  const long long tiles = cdiv(n_train, kNnTile);
  // split the training columns for the best-filled waves (resident CTAs per SM
  // from the occupancy API); a larger split must fill them by 2 points more
  static int nn_occ = 0;
  if (nn_occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nn_occ, k_nearest, kThreads, 0) != cudaSuccess ||
        nn_occ < 1)
      nn_occ = 1;
  }
  const long long slots = (long long)nn_occ * ctx->nsm;
  long long nsplit = 1, per = tiles * kNnTile;
  {
    double best_eff = 0.0;
    for (long long sp = 1; sp <= std::min<long long>(tiles, 16); ++sp) {
      const long long pr = cdiv(tiles, sp) * kNnTile;
      const long long ns = cdiv(n_train, pr);
      const long long c = gx * ns, waves = cdiv(c, slots);
      const double eff = (double)c / (double)(waves * slots);
      if (sp == 1 || eff > best_eff + 0.02) {
        best_eff = eff;
        nsplit = ns;
        per = pr;
      }
    }
  }
  if (gx > 0x7fffffffLL || nsplit > 65535)
    return set_err(RBD_ERR_INVALID_ARGUMENT, "nearest: problem too large for one launch");
  TRY(ensure(ctx->nn_part, sizeof(NnRec) * (size_t)nsplit * (size_t)Q));
  k_nearest<<<dim3((unsigned)gx, (unsigned)nsplit), kThreads, 0, ctx->stream>>>(
      dC, ldc, dT, n_train, d, Q, per, ptr<NnRec>(ctx->nn_part));
  const int gr = (int)std::max<long long>(1, std::min<long long>(cdiv(Q, 256), (long long)ctx->nsm * 4));
  k_nearest_reduce<<<gr, 256, 0, ctx->stream>>>(ptr<NnRec>(ctx->nn_part), Q, (int)nsplit,
                                                reinterpret_cast<long long*>(d_best),
                                                d_dist);
  ctx->launches += 2;
  CU(cudaGetLastError());
  return RBD_OK;
}

int rbd_classify_batch(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                       const double* dT, int64_t n_train, const double* dQ, int64_t Q,
                       int64_t ldq, int64_t* d_best, double* d_dist) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || n_train < 1 || Q < 0)
    return set_err(RBD_ERR_DIMENSION_MISMATCH, "classify: bad sizes");
  if (ldy < m || ldq < m)
    return set_err(RBD_ERR_DIMENSION_MISMATCH, "classify: test dimension != training dimension");
  if (Q == 0) return RBD_OK;
  CU(cudaSetDevice(ctx->device));
  TRY(ensure(ctx->nn_coords, sizeof(double) * (size_t)d * (size_t)Q));
  double* C = ptr<double>(ctx->nn_coords);
  TRY(rbd_project_batch(ctx, dY, m, d, ldy, dQ, Q, ldq, C, nullptr));   // c = Y'v (K5)
  return rbd_nearest_columns(ctx, C, d, Q, d, dT, n_train, d_best, d_dist);
}

int rbd_classify_host(rbd_ctx_t ctx, const double* hY, int64_t m, int64_t d, const double* hT,
                      int64_t n_train, const double* hQ, int64_t Q, int64_t* h_best,
                      double* h_dist) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || n_train < 1 || Q < 0)
    return set_err(RBD_ERR_DIMENSION_MISMATCH, "classify: bad sizes");
  if (Q == 0) return RBD_OK;
  CU(cudaSetDevice(ctx->device));
  DevBuf bY, bT, bQ, bB, bD;
  auto fin = [&](int rc) {
    release(bY);
    release(bT);
    release(bQ);
    release(bB);
    release(bD);
    return rc;
  };
  const long long ldm = (m % 2 == 0) ? m : m + 1;   // 16-byte aligned columns for K5
  int rc;
  if ((rc = ensure(bY, sizeof(double) * ldm * d)) || (rc = ensure(bT, sizeof(double) * d * n_train)) ||
      (rc = ensure(bQ, sizeof(double) * ldm * Q)) || (rc = ensure(bB, sizeof(int64_t) * Q)) ||
      (rc = ensure(bD, sizeof(double) * Q)))
    return fin(rc);
  if (cudaMemcpy2DAsync(bY.p, sizeof(double) * ldm, hY, sizeof(double) * m, sizeof(double) * m, d,
                        cudaMemcpyHostToDevice, ctx->stream) ||
      cudaMemcpyAsync(bT.p, hT, sizeof(double) * d * n_train, cudaMemcpyHostToDevice, ctx->stream) ||
      cudaMemcpy2DAsync(bQ.p, sizeof(double) * ldm, hQ, sizeof(double) * m, sizeof(double) * m, Q,
                        cudaMemcpyHostToDevice, ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "classify_host: H2D failed"));
  rc = rbd_classify_batch(ctx, ptr<double>(bY), m, d, ldm, ptr<double>(bT), n_train, ptr<double>(bQ),
                          Q, ldm, ptr<int64_t>(bB), ptr<double>(bD));
  if (rc) return fin(rc);
  if (cudaMemcpyAsync(h_best, bB.p, sizeof(int64_t) * Q, cudaMemcpyDeviceToHost, ctx->stream) ||
      (h_dist && cudaMemcpyAsync(h_dist, bD.p, sizeof(double) * Q, cudaMemcpyDeviceToHost,
                                 ctx->stream)) ||
      cudaStreamSynchronize(ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "classify_host: D2H failed"));
  return fin(RBD_OK);
}

int rbd_reconstruct(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                    const double* dc, double* dv) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (ldy < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "reconstruct: ldy < m");
  CU(cudaSetDevice(ctx->device));
  long long nl = 0;
  int rc = rbdk::launch_reconstruct_f64(dY, m, d, ldy, dc, dv, ctx->stream, &nl);
  ctx->launches += nl;
  if (rc != 0) return set_err(RBD_ERR_CUDA, std::string("reconstruct kernel: ") + cudaGetErrorString((cudaError_t)rc));
  return RBD_OK;
}

}  // extern "C"

extern "C" {

int rbd_project_host(rbd_ctx_t ctx, const double* hY, int64_t m, int64_t d, const double* hXn,
                     int64_t N, double* hTn, double* h_err) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || N < 0) return set_err(RBD_ERR_DIMENSION_MISMATCH, "project: bad sizes");
  if (N == 0) return RBD_OK;
  CU(cudaSetDevice(ctx->device));
  DevBuf bY, bX, bT, bE;
  auto fin = [&](int rc) {
    release(bY);
    release(bX);
    release(bT);
    release(bE);
    return rc;
  };
  int rc;
  if ((rc = ensure(bY, sizeof(double) * m * d)) || (rc = ensure(bX, sizeof(double) * m * N)) ||
      (rc = ensure(bT, sizeof(double) * d * N)) || (rc = ensure(bE, sizeof(double) * N)))
    return fin(rc);
  if (cudaMemcpyAsync(bY.p, hY, sizeof(double) * m * d, cudaMemcpyHostToDevice, ctx->stream) ||
      cudaMemcpyAsync(bX.p, hXn, sizeof(double) * m * N, cudaMemcpyHostToDevice, ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "project_host: H2D failed"));
  rc = rbd_project_batch(ctx, ptr<double>(bY), m, d, m, ptr<double>(bX), N, m, ptr<double>(bT),
                         h_err ? ptr<double>(bE) : nullptr);
  if (rc) return fin(rc);
  if (hTn && cudaMemcpyAsync(hTn, bT.p, sizeof(double) * d * N, cudaMemcpyDeviceToHost, ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "project_host: D2H failed"));
  if (h_err && cudaMemcpyAsync(h_err, bE.p, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "project_host: D2H failed"));
  if (cudaStreamSynchronize(ctx->stream)) return fin(set_err(RBD_ERR_CUDA, "project_host: sync failed"));
  return fin(RBD_OK);
}

int rbd_reconstruct_host(rbd_ctx_t ctx, const double* hY, int64_t m, int64_t d, const double* hc,
                         double* hv) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 0) return set_err(RBD_ERR_DIMENSION_MISMATCH, "reconstruct: bad sizes");
  CU(cudaSetDevice(ctx->device));
  DevBuf bY, bc, bv;
  auto fin = [&](int rc) {
    release(bY);
    release(bc);
    release(bv);
    return rc;
  };
  int rc;
  if ((rc = ensure(bY, sizeof(double) * m * std::max<int64_t>(d, 1))) ||
      (rc = ensure(bc, sizeof(double) * std::max<int64_t>(d, 1))) || (rc = ensure(bv, sizeof(double) * m)))
    return fin(rc);
  if (d > 0 && (cudaMemcpyAsync(bY.p, hY, sizeof(double) * m * d, cudaMemcpyHostToDevice, ctx->stream) ||
                cudaMemcpyAsync(bc.p, hc, sizeof(double) * d, cudaMemcpyHostToDevice, ctx->stream)))
    return fin(set_err(RBD_ERR_CUDA, "reconstruct_host: H2D failed"));
  rc = rbd_reconstruct(ctx, ptr<double>(bY), m, d, m, ptr<double>(bc), ptr<double>(bv));
  if (rc) return fin(rc);
  if (cudaMemcpyAsync(hv, bv.p, sizeof(double) * m, cudaMemcpyDeviceToHost, ctx->stream) ||
      cudaStreamSynchronize(ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "reconstruct_host: D2H failed"));
  return fin(RBD_OK);
}

int rbd_time_sweep(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx,
                   const double* dy, int reps, double* ms_per_launch) {
  if (!ctx || reps < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "time_sweep: bad arguments");
  CU(cudaSetDevice(ctx->device));
  TRY(ensure(ctx->partial, sizeof(double) * cdiv(m, kChunk) * n));
  const int vec = (ldx % 2 == 0 && aligned16(dX) && aligned16(dy)) ? 2 : 1;
  SweepArgs s{};
  s.A = dX;
  s.lda = ldx;
  s.m = m;
  s.ncols = n;
  s.v = dy;
  s.partial = ptr<double>(ctx->partial);
  s.pstride = n;
  s.gate = GATE_NONE;
  TRY(launch_sweep(ctx, s, vec, MODE_DOT, true, n));  // warm-up
  cudaEvent_t a, b;
  CU(cudaEventCreate(&a));
  CU(cudaEventCreate(&b));
  cudaEventRecord(a, ctx->stream);
  for (int r = 0; r < reps; ++r) {
    int rc = launch_sweep(ctx, s, vec, MODE_DOT, true, n);
    if (rc) {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      return rc;
    }
  }
  cudaEventRecord(b, ctx->stream);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (e != cudaSuccess) return set_err(RBD_ERR_CUDA, std::string("time_sweep: ") + cudaGetErrorString(e));
  *ms_per_launch = ms / reps;
  return RBD_OK;
}

}  // extern "C"

// ===========================================================================
// Sharded (multi-GPU) greedy loop — SURVEY.md §8(e)
//
// X is split by contiguous column blocks, Y is replicated. Each step every
// rank runs the one-step mode of the persistent kernel on its shard
// (k_rbd_persistent<VEC, true>): the replicated extension pass, the replicated
// Y'w1 tiles (identical bits on every rank), the local X'w1 sweep and
// finalisation, and packs a payload = (its best residual, global index,
// col_sq, x_j, T[0:k+1, j]). One allgather of payloads replaces the max-loc
// allreduce + owner broadcast (exact: no arithmetic on the data), and
// k_shard_select picks the winner identically on every rank. Per-column sums
// depend on m only, so results are bit-identical for any number of shards.
//
// Two exchanges: NCCL (one process per GPU, NCCL loaded with dlopen) and
// virtual ranks (R shards in one process on one device, stepped in lockstep on
// one stream — no kernel ever waits for another rank).
// ===========================================================================
#include <nccl.h>

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names)
      if ((a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!a.h) return a;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(a.h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(a.h, "ncclCommInitRank");
    a.AllGather = (decltype(a.AllGather))dlsym(a.h, "ncclAllGather");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(a.h, "ncclCommDestroy");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(a.h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllGather && a.CommDestroy && a.GetErrorString;
    return a;
  }();
  return api;
}

struct Exchange {
  virtual ~Exchange() = default;
  virtual int world() const = 0;
  // every rank's `count` doubles of send -> slot [rank] of every rank's recv
  virtual int allgather(std::vector<rbd_ctx_t>& R, long long count) = 0;
};

struct LocalExchange : Exchange {
  int R;
  explicit LocalExchange(int r) : R(r) {}
  int world() const override { return R; }
  int allgather(std::vector<rbd_ctx_t>& ranks, long long count) override {
    for (int r = 0; r < R; ++r)
      for (int s = 0; s < R; ++s)
        CU(cudaMemcpyAsync(ptr<double>(ranks[r]->recv) + (long long)s * count, ranks[s]->send.p,
                           sizeof(double) * count, cudaMemcpyDeviceToDevice, ranks[r]->stream));
    return RBD_OK;
  }
};

struct NcclExchange : Exchange {
  int W;
  explicit NcclExchange(int w) : W(w) {}
  int world() const override { return W; }
  int allgather(std::vector<rbd_ctx_t>& ranks, long long count) override {
    rbd_ctx_t c = ranks[0];
    ncclResult_t r = nccl().AllGather(c->send.p, c->recv.p, (size_t)count, ncclDouble,
                                      (ncclComm_t)c->comm, c->stream);
    if (r != ncclSuccess) return set_err(RBD_ERR_NCCL, std::string("ncclAllGather: ") + nccl().GetErrorString(r));
    return RBD_OK;
  }
};

struct Shard {
  const double* X;
  long long n_local;
  long long col_offset;
  double* Y;
  double* T;
};

int shard_step_launch(rbd_ctx_t c, const Shard& sh, long long m, long long ldx, long long d_max,
                      long long pay_stride, int vec, int grid) {
  PersistArgs a{};
  a.X = sh.X;
  a.ldx = ldx;
  a.m = m;
  a.n = sh.n_local;
  a.Y = sh.Y;
  a.T = sh.T;
  a.w = ptr<double>(c->w);
  a.p = ptr<double>(c->gcnt);
  a.ppart = ptr<double>(c->ppart);
  a.npart = ptr<double>(c->nrm);
  a.partial = ptr<double>(c->partial);
  a.r = ptr<double>(c->resid);
  a.col_sq = ptr<double>(c->colsq);
  a.rec = ptr<Rec>(c->ygcnt);
  a.history = ptr<double>(c->hist);
  a.selected = ptr<long long>(c->sel);
  a.st = ptr<DevState>(c->state);
  a.bar = ptr<unsigned>(c->bar);
  a.d_max = d_max;
  a.ctl = ptr<StepCtl>(c->ctl);
  a.rdy = ptr<unsigned long long>(c->rdy);
  a.recv = ptr<double>(c->recv);
  a.send = ptr<double>(c->send);
  a.pay_stride = pay_stride;
  a.col_offset = sh.col_offset;
  void* args[] = {&a};
  const size_t smem = persist_smem(d_max);
  cudaError_t e = vec == 2 ? cudaLaunchCooperativeKernel((void*)k_rbd_persistent<2, true>, grid,
                                                         kThreads, args, smem, c->stream)
                           : cudaLaunchCooperativeKernel((void*)k_rbd_persistent<1, true>, grid,
                                                         kThreads, args, smem, c->stream);
  c->launches++;
  if (e != cudaSuccess)
    return set_err(RBD_ERR_CUDA, std::string("sharded step launch: ") + cudaGetErrorString(e));
  return RBD_OK;
}

int sharded_decompose(std::vector<rbd_ctx_t>& R, Exchange& ex, std::vector<Shard>& sh, long long m,
                      long long ldx, long long n_global, const rbd_config_t* cfg,
                      int64_t* h_selected, double* h_history, rbd_result_t* result) {
  if (m < 1 || n_global < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: matrix must be non-empty");
  const int nl = (int)R.size();
  const long long d_cap = std::max<long long>(1, std::min<long long>(cfg->d_max, n_global));
  if (d_cap > kFMaxCoef)
    return set_err(RBD_ERR_INVALID_ARGUMENT, "sharded decompose: d_max above the fused-path limit");
  const long long pay_stride = ((kPayHead + m + d_cap + 1) + 1) / 2 * 2;
  bool vec2 = (ldx % 2 == 0) && (m % 2 == 0);
  for (auto& s : sh) vec2 = vec2 && aligned16(s.X) && aligned16(s.Y);
  const int vec = vec2 ? 2 : 1;
  // ---- K1 on every shard, then a global combine of (finite, nonzero, max col_sq) ----
  for (int r = 0; r < nl; ++r) {
    rbd_ctx_t c = R[r];
    CU(cudaSetDevice(c->device));
    const long long nloc = std::max<long long>(sh[r].n_local, 1);
    TRY(ensure_loop_buffers(c, m, nloc, d_cap));
    TRY(ensure(c->send, sizeof(double) * pay_stride));
    TRY(ensure(c->recv, sizeof(double) * pay_stride * ex.world()));
    TRY(ensure(c->ctl, sizeof(StepCtl)));
    TRY(ensure(c->gcnt, sizeof(double) * 2 * (size_t)(d_cap + 1)));
    TRY(ensure(c->rdy, sizeof(unsigned long long) * (size_t)(cdiv(m, kChunk) + 1)));
    const int grid = persistent_grid(c, vec, d_cap);
    TRY(ensure(c->ppart, sizeof(double) * (size_t)std::max<long long>(grid, cdiv(m, kChunk)) * d_cap));
    TRY(ensure(c->nrm, sizeof(double) * std::max<long long>(gemv_grid(m), grid)));
    TRY(ensure(c->ygcnt, sizeof(Rec) * (size_t)grid));
    DevState* st = ptr<DevState>(c->state);
    CU(cudaMemsetAsync(st, 0, sizeof(DevState), c->stream));
    CU(cudaMemsetAsync(c->ctl.p, 0, sizeof(StepCtl), c->stream));
    CU(cudaMemsetAsync(c->rdy.p, 0, sizeof(unsigned long long) * (size_t)(cdiv(m, kChunk) + 1),
                       c->stream));
    CU(cudaMemsetAsync(c->bar.p, 0, 64, c->stream));
    CU(cudaMemsetAsync(c->partial.p, 0xFF, sizeof(double) * (size_t)cdiv(m, kChunk) * nloc, c->stream));
    if (sh[r].n_local > 0)
      TRY(enqueue_init(c, sh[r].X, m, sh[r].n_local, ldx, ptr<double>(c->partial),
                       ptr<double>(c->colsq), ptr<double>(c->resid), st));
    CU(cudaMemsetAsync(c->partial.p, 0xFF, sizeof(double) * (size_t)cdiv(m, kChunk) * nloc, c->stream));
    CU(cudaMemsetAsync(c->counter.p, 0, 64, c->stream));
    CU(cudaMemcpyAsync(c->h_state, st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    double head[4] = {(double)c->h_state->flags_nonfinite, (double)c->h_state->flags_nonzero, 0.0, 0.0};
    std::memcpy(&head[2], &c->h_state->max_colsq_bits, sizeof(double));
    CU(cudaMemcpyAsync(c->send.p, head, sizeof(head), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));   // head is a stack buffer
  }
  TRY(ex.allgather(R, 4));
  std::vector<double> all(4 * (size_t)ex.world());
  CU(cudaMemcpyAsync(all.data(), R[0]->recv.p, sizeof(double) * all.size(), cudaMemcpyDeviceToHost,
                     R[0]->stream));
  CU(cudaStreamSynchronize(R[0]->stream));
  DevState hs{};
  double max_colsq = 0.0;
  for (int w = 0; w < ex.world(); ++w) {
    hs.flags_nonfinite |= all[4 * w] != 0.0;
    hs.flags_nonzero |= all[4 * w + 1] != 0.0;
    max_colsq = std::max(max_colsq, all[4 * w + 2]);
  }
  TRY(validate_after_init(cfg, m, n_global, hs));
  const double tol = breakdown_tolerance(cfg, m, max_colsq);
  long long j0 = 0;
  TRY(start_column(cfg, n_global, &j0));
  // ---- loop state + seed exchange (the owner of the start column publishes it) ----
  for (int r = 0; r < nl; ++r) {
    rbd_ctx_t c = R[r];
    DevState s0{};
    s0.d = 0;
    s0.jstar = j0;
    s0.d_max = cfg->d_max;
    s0.e_cur = std::numeric_limits<double>::infinity();
    s0.eps_R = cfg->eps_R;
    s0.breakdown_tol = tol;
    s0.done = !(0 < cfg->d_max && s0.e_cur > cfg->eps_R) ? 1 : 0;
    s0.cfg_reorth = cfg->reorthogonalize ? 1 : 0;
    s0.wnorm = 1.0;
    *c->h_state = s0;
    CU(cudaMemcpyAsync(c->state.p, c->h_state, sizeof(DevState), cudaMemcpyHostToDevice, c->stream));
    const long long jl = (j0 >= sh[r].col_offset && j0 < sh[r].col_offset + sh[r].n_local)
                             ? j0 - sh[r].col_offset : -1;
    k_shard_seed_pack<<<64, 256, 0, c->stream>>>(sh[r].X, ldx, m, jl, sh[r].col_offset,
                                                 ptr<double>(c->colsq), ptr<double>(c->send));
    c->launches++;
    CU(cudaStreamSynchronize(c->stream));   // pinned h_state reused below
  }
  TRY(ex.allgather(R, pay_stride));
  for (int r = 0; r < nl; ++r) {
    k_shard_seed_select<<<1, 32, 0, R[r]->stream>>>(ptr<DevState>(R[r]->state), ptr<double>(R[r]->recv),
                                                    pay_stride, ex.world());
    R[r]->launches++;
  }
  // ---- greedy loop: step kernels, payload allgather, winner selection ----
  std::vector<int> grids(nl);
  for (int r = 0; r < nl; ++r) grids[r] = persistent_grid(R[r], vec, d_cap);
  for (long long step = 0; step < cfg->d_max; ++step) {
    for (int r = 0; r < nl; ++r)
      TRY(shard_step_launch(R[r], sh[r], m, ldx, d_cap, pay_stride, vec, grids[r]));
    TRY(ex.allgather(R, pay_stride));
    for (int r = 0; r < nl; ++r) {
      k_shard_select<<<1, 32, 0, R[r]->stream>>>(ptr<DevState>(R[r]->state), ptr<double>(R[r]->recv),
                                                 pay_stride, ex.world(), ptr<double>(R[r]->hist),
                                                 ptr<long long>(R[r]->sel));
      R[r]->launches++;
    }
    CU(cudaGetLastError());
    if ((step & 3) == 3 || step + 1 == cfg->d_max) {
      CU(cudaMemcpyAsync((void*)&R[0]->h_state->done, &ptr<DevState>(R[0]->state)->done, sizeof(int),
                         cudaMemcpyDeviceToHost, R[0]->stream));
      CU(cudaStreamSynchronize(R[0]->stream));
      if (R[0]->h_state->done) break;
    }
  }
  // the last accepted column's second pass
  for (int r = 0; r < nl; ++r) TRY(shard_step_launch(R[r], sh[r], m, ldx, d_cap, pay_stride, vec, grids[r]));
  for (int r = 0; r < nl; ++r) CU(cudaStreamSynchronize(R[r]->stream));
  rbd_ctx_t c0 = R[0];
  CU(cudaMemcpy(c0->h_state, c0->state.p, sizeof(DevState), cudaMemcpyDeviceToHost));
  const long long d = c0->h_state->d;
  if (d == 0)
    return set_err(RBD_ERR_DEGENERATE_INPUT, "decompose: start column is numerically zero, no basis built");
  if (h_selected) CU(cudaMemcpy(h_selected, c0->sel.p, sizeof(long long) * d, cudaMemcpyDeviceToHost));
  if (h_history) CU(cudaMemcpy(h_history, c0->hist.p, sizeof(double) * d, cudaMemcpyDeviceToHost));
  if (result) {
    result->d = d;
    result->breakdown = c0->h_state->breakdown;
    result->breakdown_tol = tol;
    result->max_col_norm = std::sqrt(max_colsq);
    result->launches = 0;
    for (auto c : R) result->launches += c->launches;
  }
  return RBD_OK;
}

}  // namespace

void rbd_comm_release(rbd_ctx_t ctx) {
  if (ctx && ctx->comm && nccl().ok) {
    nccl().CommDestroy((ncclComm_t)ctx->comm);
    ctx->comm = nullptr;
  }
}

extern "C" {

int rbd_comm_unique_id(char out[RBD_UNIQUE_ID_BYTES]) {
  if (!nccl().ok) return set_err(RBD_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded");
  ncclUniqueId id;
  ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) return set_err(RBD_ERR_NCCL, std::string("ncclGetUniqueId: ") + nccl().GetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == RBD_UNIQUE_ID_BYTES, "unique id size");
  std::memcpy(out, &id, RBD_UNIQUE_ID_BYTES);
  return RBD_OK;
}

int rbd_ctx_init_comm(rbd_ctx_t ctx, int rank, int world, const char id[RBD_UNIQUE_ID_BYTES]) {
  if (!ctx || world < 1 || rank < 0 || rank >= world)
    return set_err(RBD_ERR_INVALID_ARGUMENT, "init_comm: bad rank/world");
  if (!nccl().ok) return set_err(RBD_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded");
  CU(cudaSetDevice(ctx->device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, RBD_UNIQUE_ID_BYTES);
  ncclComm_t comm;
  ncclResult_t r = nccl().CommInitRank(&comm, world, uid, rank);
  if (r != ncclSuccess) return set_err(RBD_ERR_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
  rbd_comm_release(ctx);
  ctx->comm = comm;
  ctx->rank = rank;
  ctx->world = world;
  return RBD_OK;
}

int rbd_decompose_sharded(rbd_ctx_t ctx, const double* dX_local, int64_t m, int64_t n_local,
                          int64_t ldx, int64_t col_offset, int64_t n_global,
                          const rbd_config_t* cfg, double* dY, double* dT_local,
                          int64_t* h_selected, double* h_history, rbd_result_t* result) {
  if (!ctx || !cfg) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: null context/config");
  if (!ctx->comm) return set_err(RBD_ERR_NCCL, "sharded decompose: call rbd_ctx_init_comm first");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "decompose: ldx < m");
  std::vector<rbd_ctx_t> R{ctx};
  std::vector<Shard> sh{Shard{dX_local, n_local, col_offset, dY, dT_local}};
  NcclExchange ex(ctx->world);
  return sharded_decompose(R, ex, sh, m, ldx, n_global, cfg, h_selected, h_history, result);
}

int rbd_decompose_sharded_virtual(rbd_ctx_t ctx, int nranks, const double* const* dX_shards,
                                  const int64_t* n_locals, int64_t m, int64_t ldx,
                                  const rbd_config_t* cfg, double* const* dY_ranks,
                                  double* const* dT_ranks, int64_t* h_selected, double* h_history,
                                  rbd_result_t* result) {
  if (!ctx || !cfg || nranks < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "virtual sharded: bad arguments");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "decompose: ldx < m");
  CU(cudaSetDevice(ctx->device));
  while ((int)ctx->virt.size() < nranks) {
    auto* sub = new rbd_ctx_s();
    sub->device = ctx->device;
    sub->nsm = ctx->nsm;
    sub->occ_sweep2 = ctx->occ_sweep2;
    sub->occ_sweep1 = ctx->occ_sweep1;
    sub->fused_grid_cap = ctx->fused_grid_cap;
    sub->stream = ctx->stream;
    cudaMallocHost(&sub->h_state, sizeof(DevState));
    cudaMallocHost(&sub->h_rec, sizeof(Rec) * 4);
    if (ensure(sub->bar, 64) == RBD_OK) cudaMemset(sub->bar.p, 0, 64);
    ctx->virt.push_back(sub);
  }
  std::vector<rbd_ctx_t> R(ctx->virt.begin(), ctx->virt.begin() + nranks);
  for (auto c : R) c->stream = ctx->stream;
  std::vector<Shard> sh(nranks);
  long long off = 0;
  for (int r = 0; r < nranks; ++r) {
    sh[r] = Shard{dX_shards[r], n_locals[r], off, dY_ranks[r], dT_ranks[r]};
    off += n_locals[r];
  }
  LocalExchange ex(nranks);
  const long long l0 = 0;
  for (auto c : R) c->launches = l0;
  int rc = sharded_decompose(R, ex, sh, m, ldx, off, cfg, h_selected, h_history, result);
  for (auto c : R) ctx->launches += c->launches;
  return rc;
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
  DevBuf bv, bB, bx;
  auto fin = [&](int rc) {
    release(bv);
    release(bB);
    release(bx);
    return rc;
  };
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

int rbd_ws_init_host(rbd_ctx_t ctx, const double* hX, int64_t m, int64_t n, int64_t ldx,
                     int64_t cap, rbd_ws_t* out) {
  if (!ctx || !out) return set_err(RBD_ERR_INVALID_ARGUMENT, "null argument");
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "workspace_init: empty matrix");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "workspace_init: ldx < m");
  CU(cudaSetDevice(ctx->device));
  DevBuf xb;
  TRY(ensure(xb, sizeof(double) * m * n));
  if (cudaMemcpy2DAsync(xb.p, sizeof(double) * m, hX, sizeof(double) * ldx, sizeof(double) * m, n,
                        cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess) {
    release(xb);
    return set_err(RBD_ERR_CUDA, "workspace_init: H2D failed");
  }
  rbd_ws_t ws = nullptr;
  int rc = rbd_ws_init(ctx, ptr<double>(xb), m, n, m, cap, &ws);
  if (rc) {
    release(xb);
    return rc;
  }
  ws->Xown = xb;
  *out = ws;
  return RBD_OK;
}

int rbd_ws_init_diag_host(rbd_ctx_t ctx, const double* hX, int64_t m, int64_t n, int64_t ldx,
                          int64_t cap, const double* h_diag, int64_t diag_len, rbd_ws_t* out) {
  if (!ctx || !out) return set_err(RBD_ERR_INVALID_ARGUMENT, "null argument");
  TRY(check_diagonal(h_diag, diag_len));
  if (m < 1 || n < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "workspace_init: empty matrix");
  if (ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "workspace_init: ldx < m");
  if (diag_len != m)
    return set_err(RBD_ERR_INCOMPATIBLE_WEIGHT, "weight dimension does not match matrix rows");
  CU(cudaSetDevice(ctx->device));
  DevBuf xb, db;
  TRY(ensure(xb, sizeof(double) * m * n));
  if (ensure(db, sizeof(double) * m) != RBD_OK ||
      cudaMemcpy2DAsync(xb.p, sizeof(double) * m, hX, sizeof(double) * ldx, sizeof(double) * m, n,
                        cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
      cudaMemcpyAsync(db.p, h_diag, sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream) !=
          cudaSuccess) {
    release(xb);
    release(db);
    return set_err(RBD_ERR_CUDA, "workspace_init: H2D failed");
  }
  rbd_ws_t ws = nullptr;
  int rc = rbd_ws_init_diag(ctx, ptr<double>(xb), m, n, m, cap, ptr<double>(db), m, &ws);
  release(db);   // the workspace keeps its own copy of the weight
  if (rc) {
    release(xb);
    return rc;
  }
  ws->Xown = xb;
  *out = ws;
  return RBD_OK;
}

int rbd_ws_extend_host(rbd_ws_t ws, const double* hxi) {
  if (!ws) return set_err(RBD_ERR_INVALID_ARGUMENT, "null workspace");
  DevBuf b;
  TRY(ensure(b, sizeof(double) * ws->m));
  // on the workspace's stream (a pageable-source cudaMemcpy may return before its
  // DMA lands, and the context stream does not wait for the legacy stream)
  if (cudaMemcpyAsync(b.p, hxi, sizeof(double) * ws->m, cudaMemcpyHostToDevice,
                      ws->ctx->stream) != cudaSuccess) {
    release(b);
    return set_err(RBD_ERR_CUDA, "workspace_extend: H2D failed");
  }
  int rc = rbd_ws_extend(ws, ptr<double>(b));
  release(b);
  return rc;
}

int rbd_reconstruct_batch(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                          const double* dC, int64_t N, double* dV) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (ldy < m || m < 1 || N < 0) return set_err(RBD_ERR_DIMENSION_MISMATCH, "compress: bad sizes");
  if (N == 0) return RBD_OK;
  CU(cudaSetDevice(ctx->device));
  if (d >= 1 && launch_compress_dmma<true>(dY, m, d, ldy, dC, N, d, dV, m, ctx->stream)) {
    ctx->launches += cdiv(cdiv(N, 64), 65535);
    CU(cudaGetLastError());
    return RBD_OK;
  }
  const long long gx = std::min<long long>(cdiv(m, 256), 1024);
  for (long long j0 = 0; j0 < N; j0 += 65535) {
    const long long nb = std::min<long long>(65535, N - j0);
    k_reconstruct_batch<<<dim3((unsigned)gx, (unsigned)nb), 256, 0, ctx->stream>>>(
        dY, m, d, ldy, dC + j0 * d, nb, dV + j0 * m);
    ctx->launches++;
  }
  CU(cudaGetLastError());
  return RBD_OK;
}

int rbd_compress_device(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                        const double* dT, int64_t n, int64_t ldt, double* dV, int64_t ldv) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || n < 0 || ldy < m || ldt < n || ldv < m)
    return set_err(RBD_ERR_DIMENSION_MISMATCH, "compress: bad sizes");
  if (n == 0) return RBD_OK;
  CU(cudaSetDevice(ctx->device));
  if (launch_compress_dmma<false>(dY, m, d, ldy, dT, n, ldt, dV, ldv, ctx->stream)) {
    ctx->launches += cdiv(cdiv(n, 64), 65535);
    CU(cudaGetLastError());
    return RBD_OK;
  }
  // unaligned operands: transpose T into column-major coefficients, SIMT path
  DevBuf c;
  TRY(ensure(c, sizeof(double) * (size_t)d * (size_t)n));
  for (int64_t k = 0; k < d; ++k)   // row k of T -> element k of every column
    CU(cudaMemcpy2DAsync(ptr<double>(c) + k, sizeof(double) * d, dT + k * ldt, sizeof(double),
                         sizeof(double), n, cudaMemcpyDeviceToDevice, ctx->stream));
  int rc = RBD_OK;
  if (ldv == m) {
    rc = rbd_reconstruct_batch(ctx, dY, m, d, ldy, ptr<double>(c), n, dV);
  } else {
    rc = set_err(RBD_ERR_INVALID_ARGUMENT, "compress: unaligned operands need ldv == m");
  }
  cudaStreamSynchronize(ctx->stream);
  release(c);
  return rc;
}

int rbd_compress_host(rbd_ctx_t ctx, const double* hY, int64_t m, int64_t d, const double* hC,
                      int64_t N, double* hV) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || N < 1) return set_err(RBD_ERR_DIMENSION_MISMATCH, "compress: bad sizes");
  CU(cudaSetDevice(ctx->device));
  DevBuf bY, bC, bV;
  auto fin = [&](int rc) {
    release(bY);
    release(bC);
    release(bV);
    return rc;
  };
  int rc;
  if ((rc = ensure(bY, sizeof(double) * m * d)) || (rc = ensure(bC, sizeof(double) * d * N)) ||
      (rc = ensure(bV, sizeof(double) * m * N)))
    return fin(rc);
  if (cudaMemcpyAsync(bY.p, hY, sizeof(double) * m * d, cudaMemcpyHostToDevice, ctx->stream) ||
      cudaMemcpyAsync(bC.p, hC, sizeof(double) * d * N, cudaMemcpyHostToDevice, ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "compress_host: H2D failed"));
  rc = rbd_reconstruct_batch(ctx, ptr<double>(bY), m, d, m, ptr<double>(bC), N, ptr<double>(bV));
  if (rc) return fin(rc);
  if (cudaMemcpyAsync(hV, bV.p, sizeof(double) * m * N, cudaMemcpyDeviceToHost, ctx->stream) ||
      cudaStreamSynchronize(ctx->stream))
    return fin(set_err(RBD_ERR_CUDA, "compress_host: D2H failed"));
  return fin(RBD_OK);
}

}  // extern "C"

// ===========================================================================
// fp32 out-of-sample compression on tcgen05 (K6)
// ===========================================================================
namespace {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D fp32 column-major operand (rows = contiguous dim of length `inner`,
// `outer` columns, leading dimension ld), box 32 x 128, 128-byte swizzle.
int make_map_f32(CUtensorMap* map, const float* base, long long inner, long long outer, long long ld) {
  auto enc = tensor_map_encoder();
  if (!enc) return set_err(RBD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)kTcBK, (cuuint32_t)kTcBM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(RBD_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return RBD_OK;
}

}  // namespace

extern "C" {

int rbd_project_batch_f32(rbd_ctx_t ctx, const float* dY, int64_t m, int64_t d, int64_t ldy,
                          const float* dXn, int64_t N, int64_t ldx, float* dTn, double* d_err) {
  if (!ctx) return set_err(RBD_ERR_INVALID_ARGUMENT, "null context");
  if (m < 1 || d < 1 || N < 0) return set_err(RBD_ERR_DIMENSION_MISMATCH, "project: bad sizes");
  if (ldy < m || ldx < m) return set_err(RBD_ERR_DIMENSION_MISMATCH, "project: vector length != m");
  if (N == 0) return RBD_OK;
  if ((ldy % 4) || (ldx % 4) || !aligned16(dY) || !aligned16(dXn))
    return set_err(RBD_ERR_INVALID_ARGUMENT,
                   "project f32: leading dimensions must be multiples of 4 floats and bases 16-byte aligned (TMA)");
  CU(cudaSetDevice(ctx->device));
  CUtensorMap mY, mX;
  TRY(make_map_f32(&mY, dY, m, d, ldy));
  TRY(make_map_f32(&mX, dXn, m, N, ldx));
  static bool attr = false;
  if (!attr) {
    CU(cudaFuncSetAttribute(k_project_tf32x3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem));
    attr = true;
  }
  double* xn = nullptr;
  if (d_err) {
    TRY(ensure(ctx->scratch1, sizeof(double) * (size_t)std::max<int64_t>(N, 32)));
    xn = ptr<double>(ctx->scratch1);
  }
  // split-K over the k-blocks for the best-filled waves (1 CTA per SM): 2 for C4's 4 x 128 tiles
  const long long nk = cdiv(m, kTcBK);
  const long long ctas = cdiv(d, kTcBM) * cdiv(N, kTcBN);
  int sk = 1;
  {
    double best_eff = 0.0;
    for (int s = 1; s <= 4; ++s) {
      if (s > 1 && nk / s < 64) break;
      const long long c = ctas * s, waves = cdiv(c, ctx->nsm);
      const double eff = (double)c / (double)(waves * ctx->nsm);
      if (s == 1 || eff > best_eff + 0.02) {
        sk = s;
        best_eff = eff;
      }
    }
  }
  const int kb_per = (int)cdiv(nk, sk);
  sk = (int)cdiv(nk, kb_per);   // every split gets at least one k-block
  float* Tws = nullptr;
  double* xws = nullptr;
  if (sk > 1) {
    const size_t tbytes = sizeof(float) * (size_t)(sk - 1) * (size_t)(d * N);
    TRY(ensure(ctx->pj_ws, tbytes + sizeof(double) * (size_t)(sk - 1) * (size_t)N + 16));
    Tws = ptr<float>(ctx->pj_ws);
    xws = reinterpret_cast<double*>(reinterpret_cast<char*>(ctx->pj_ws.p) + ((tbytes + 15) & ~(size_t)15));
  }
  dim3 grid((unsigned)cdiv(d, kTcBM), (unsigned)cdiv(N, kTcBN), (unsigned)sk);
  k_project_tf32x3<<<grid, kTcThreads, kTcSmem, ctx->stream>>>(mY, mX, m, d, N, dTn, xn, kb_per,
                                                                Tws, xws);
  ctx->launches++;
  CU(cudaGetLastError());
  if (sk > 1) {
    k_splitk_sum_f32<<<1184, 256, 0, ctx->stream>>>(dTn, Tws, d * N, sk - 1, xn, xws, N);
    ctx->launches++;
    CU(cudaGetLastError());
  }
  if (d_err) {
    k_project_err_f32<<<(unsigned)cdiv(N, 8), 256, 0, ctx->stream>>>(xn, dTn, d, N, d_err);
    ctx->launches++;
    CU(cudaGetLastError());
  }
  return RBD_OK;
}

}  // extern "C"
