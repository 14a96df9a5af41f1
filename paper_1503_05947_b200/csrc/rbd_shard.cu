// rbd_shard.cu — the multi-GPU (column-sharded) greedy loop behind the C ABI
// (SURVEY §8(e)): NCCL payload exchange and virtual ranks.
#include "rbd_capi_internal.h"
#include "rbd_persistent.cuh"

// ===========================================================================
// Sharded (multi-GPU) greedy loop — SURVEY.md §8(e)
//
// X is split by contiguous column blocks, Y is replicated. A step on every
// rank (one process per GPU):
//   1. k_rbd_persistent<VEC, true> (one step per launch): the replicated
//      extension pass and Y'w1 groups (identical bits on every rank), the local
//      X'w1 sweep + finalisation, and this rank's 16-byte record {best
//      residual, global index};
//   2. ncclAllGather of the records (16 B per rank);
//   3. k_shard_pack: every rank applies the same winner rule (rbd_select.h:
//      value desc, global index asc — the reference's strict '>' scan,
//      workspace.cpp:107-113); the owner writes {col_sq, x_j, T[0:k+1, j]},
//      every other rank -0.0;
//   4. ncclAllReduce(sum) of that payload: x + -0.0 == x exactly, so every rank
//      receives the owner's bits (a max-loc + owner broadcast whose owner is
//      only known on the device);
//   5. k_shard_select: the step's bookkeeping, identical on every rank.
// The sequence is captured for kShardGraphSteps steps in a CUDA graph and
// replayed (the done flag is read one replay behind; steps after the stop are
// no-ops), so the host issues one graph launch per kShardGraphSteps steps.
// Per-column sums depend on m only: results are bit-identical for any number
// of shards. Virtual ranks (R shards on one device, lockstep on one stream,
// exchanges by device copies and an in-order sum kernel) run the same
// kernels and protocol for single-GPU tests.
// ===========================================================================
#include <nccl.h>

namespace {

constexpr int kShardGraphSteps = 8;

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
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
    a.AllReduce = (decltype(a.AllReduce))dlsym(a.h, "ncclAllReduce");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(a.h, "ncclCommDestroy");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(a.h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllGather && a.AllReduce && a.CommDestroy &&
           a.GetErrorString;
    return a;
  }();
  return api;
}

struct Exchange {
  virtual ~Exchange() = default;
  virtual int world() const = 0;
  // every rank's `count` doubles of srec -> slot [rank] of every rank's rrec
  virtual int allgather_rec(std::vector<rbd_ctx_t>& R, long long count) = 0;
  // sum over ranks of `count` doubles of send -> every rank's recv
  virtual int allreduce_pay(std::vector<rbd_ctx_t>& R, long long count) = 0;
};

struct LocalExchange : Exchange {
  int R;
  explicit LocalExchange(int r) : R(r) {}
  int world() const override { return R; }
  int allgather_rec(std::vector<rbd_ctx_t>& ranks, long long count) override {
    for (int r = 0; r < R; ++r)
      for (int s = 0; s < R; ++s)
        CU(cudaMemcpyAsync(ptr<double>(ranks[r]->rrec) + (long long)s * count, ranks[s]->srec.p,
                           sizeof(double) * count, cudaMemcpyDeviceToDevice, ranks[r]->stream));
    return RBD_OK;
  }
  int allreduce_pay(std::vector<rbd_ctx_t>& ranks, long long count) override {
    PayPtrs p{};
    for (int r = 0; r < R; ++r) {
      p.in[r] = ptr<double>(ranks[r]->send);
      p.out[r] = ptr<double>(ranks[r]->recv);
    }
    k_sum_payloads<<<(unsigned)std::max<long long>(1, std::min<long long>(cdiv(count, 256), 1184)),
                     256, 0, ranks[0]->stream>>>(p, R, count);
    ranks[0]->launches++;
    CU(cudaGetLastError());
    return RBD_OK;
  }
};

struct NcclExchange : Exchange {
  int W;
  explicit NcclExchange(int w) : W(w) {}
  int world() const override { return W; }
  int allgather_rec(std::vector<rbd_ctx_t>& ranks, long long count) override {
    rbd_ctx_t c = ranks[0];
    ncclResult_t r = nccl().AllGather(c->srec.p, c->rrec.p, (size_t)count, ncclDouble,
                                      (ncclComm_t)c->comm, c->stream);
    if (r != ncclSuccess) return set_err(RBD_ERR_NCCL, std::string("ncclAllGather: ") + nccl().GetErrorString(r));
    return RBD_OK;
  }
  int allreduce_pay(std::vector<rbd_ctx_t>& ranks, long long count) override {
    rbd_ctx_t c = ranks[0];
    ncclResult_t r = nccl().AllReduce(c->send.p, c->recv.p, (size_t)count, ncclDouble, ncclSum,
                                      (ncclComm_t)c->comm, c->stream);
    if (r != ncclSuccess) return set_err(RBD_ERR_NCCL, std::string("ncclAllReduce: ") + nccl().GetErrorString(r));
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
  a.recv = ptr<double>(c->recv);   // the winner's payload
  a.send = ptr<double>(c->srec);   // this rank's record
  a.pay_stride = pay_stride;
  a.col_offset = sh.col_offset;
  a.ydelay = y_delay(grid);
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

// One step on every rank: the step kernel, the record allgather, the pack,
// the payload allreduce and the select (see the header).
int enqueue_shard_step(std::vector<rbd_ctx_t>& R, Exchange& ex, std::vector<Shard>& sh, long long m,
                       long long ldx, long long d_cap, long long pay_stride, int vec,
                       const std::vector<int>& grids, const std::vector<int>& ranks_id) {
  const int nl = (int)R.size();
  for (int r = 0; r < nl; ++r)
    TRY(shard_step_launch(R[r], sh[r], m, ldx, d_cap, pay_stride, vec, grids[r]));
  TRY(ex.allgather_rec(R, 2));
  for (int r = 0; r < nl; ++r) {
    rbd_ctx_t c = R[r];
    k_shard_pack<<<(unsigned)std::min<long long>(cdiv(pay_stride, 256), 2 * c->nsm), 256, 0, c->stream>>>(
        ptr<DevState>(c->state), ptr<double>(c->rrec), ex.world(), ranks_id[r], sh[r].X, ldx, m,
        sh[r].T, std::max<long long>(sh[r].n_local, 1), ptr<double>(c->colsq), ptr<double>(c->send),
        pay_stride);
    c->launches++;
  }
  TRY(ex.allreduce_pay(R, pay_stride));
  for (int r = 0; r < nl; ++r) {
    rbd_ctx_t c = R[r];
    k_shard_select<<<1, 32, 0, c->stream>>>(ptr<DevState>(c->state), ptr<double>(c->rrec),
                                            ptr<double>(c->recv), ex.world(), ptr<double>(c->hist),
                                            ptr<long long>(c->sel));
    c->launches++;
  }
  CU(cudaGetLastError());
  return RBD_OK;
}

int sharded_decompose(std::vector<rbd_ctx_t>& R, Exchange& ex, std::vector<Shard>& sh, long long m,
                      long long ldx, long long n_global, const rbd_config_t* cfg,
                      int64_t* h_selected, double* h_history, rbd_result_t* result,
                      const std::vector<int>& ranks_id) {
  if (m < 1 || n_global < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "decompose: matrix must be non-empty");
  NvtxRange nv("rbd.decompose_sharded");
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
    TRY(ensure(c->recv, sizeof(double) * pay_stride));
    TRY(ensure(c->srec, sizeof(double) * 4));
    TRY(ensure(c->rrec, sizeof(double) * 4 * ex.world()));
    TRY(ensure(c->ctl, sizeof(StepCtl)));
    TRY(ensure(c->gcnt, sizeof(double) * 2 * (size_t)(d_cap + 1)));
    TRY(ensure(c->rdy, sizeof(unsigned long long) * (size_t)(cdiv(m, kChunk) + 1)));
    const int grid = persistent_grid(c, vec, d_cap);
    TRY(ensure(c->ppart, sizeof(double) * (size_t)std::max<long long>(grid, cdiv(m, kChunk)) * d_cap));
    TRY(ensure(c->nrm, sizeof(double) * std::max<long long>(gemv_grid(m), grid)));
    TRY(ensure(c->ygcnt, sizeof(Rec) * (size_t)grid));
    if (!c->h_done) CU(cudaMallocHost(&c->h_done, sizeof(double) * 4));
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
    CU(cudaMemcpyAsync(c->srec.p, head, sizeof(head), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));   // head is a stack buffer
  }
  TRY(ex.allgather_rec(R, 4));
  std::vector<double> all(4 * (size_t)ex.world());
  CU(cudaMemcpyAsync(all.data(), R[0]->rrec.p, sizeof(double) * all.size(), cudaMemcpyDeviceToHost,
                     R[0]->stream));
  CU(cudaStreamSynchronize(R[0]->stream));
  DevState hs{};
  double max_colsq = 0.0;
  for (int w = 0; w < ex.world(); ++w) {
    hs.flags_nonfinite |= all[4 * w] != 0.0;
    hs.flags_nonzero |= all[4 * w + 1] != 0.0;
    const double v = all[4 * w + 2];
    max_colsq = (std::isfinite(v) && std::isfinite(max_colsq)) ? std::max(max_colsq, v)
                                                               : INFINITY;
  }
  std::memcpy(&hs.max_colsq_bits, &max_colsq, sizeof(double));
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
    k_shard_seed_pack<<<(unsigned)std::min<long long>(cdiv(pay_stride, 256), 2 * c->nsm), 256, 0,
                        c->stream>>>(sh[r].X, ldx, m, jl, ptr<double>(c->colsq), ptr<double>(c->send),
                                     pay_stride);
    c->launches++;
    CU(cudaStreamSynchronize(c->stream));   // pinned h_state reused below
  }
  TRY(ex.allreduce_pay(R, pay_stride));
  for (int r = 0; r < nl; ++r) {
    k_shard_seed_select<<<1, 32, 0, R[r]->stream>>>(ptr<DevState>(R[r]->state), ptr<double>(R[r]->recv));
    R[r]->launches++;
  }
  // ---- greedy loop: kShardGraphSteps steps per graph replay (eager fallback) ----
  std::vector<int> grids(nl);
  for (int r = 0; r < nl; ++r) grids[r] = persistent_grid(R[r], vec, d_cap);
  const char* ge = getenv("RBD_SHARD_GRAPH");
  bool use_graph = !(ge && ge[0] == '0');
  cudaGraphExec_t gexec = nullptr;
  long long graph_launches = 0;
  if (use_graph) {
    // every virtual rank shares one stream; NCCL ranks have one context each
    cudaStream_t s0 = R[0]->stream;
    std::vector<long long> before(nl);
    for (int r = 0; r < nl; ++r) before[r] = R[r]->launches;
    cudaGraph_t g = nullptr;
    int rc = RBD_OK;
    if (cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      use_graph = false;
    } else {
      for (int s = 0; s < kShardGraphSteps && rc == RBD_OK; ++s)
        rc = enqueue_shard_step(R, ex, sh, m, ldx, d_cap, pay_stride, vec, grids, ranks_id);
      const cudaError_t ec = cudaStreamEndCapture(s0, &g);
      if (rc != RBD_OK || ec != cudaSuccess || !g ||
          cudaGraphInstantiate(&gexec, g, 0) != cudaSuccess) {
        cudaGetLastError();
        use_graph = false;
        gexec = nullptr;
      }
      if (g) cudaGraphDestroy(g);
    }
    for (int r = 0; r < nl; ++r) {
      graph_launches += R[r]->launches - before[r];
      R[r]->launches = before[r];   // counted per replay below
    }
    if (!use_graph && rc == RBD_OK) set_err(RBD_OK, "");
  }
  if (use_graph) {
    struct GraphGuard {
      cudaGraphExec_t g;
      ~GraphGuard() {
        if (g) cudaGraphExecDestroy(g);
      }
    } guard{gexec};
    cudaEvent_t ev[2];
    CU(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    struct EvGuard {
      cudaEvent_t* e;
      ~EvGuard() {
        cudaEventDestroy(e[0]);
        cudaEventDestroy(e[1]);
      }
    } eg{ev};
    rbd_ctx_t c0 = R[0];
    int* hd = reinterpret_cast<int*>(c0->h_done);
    hd[0] = hd[1] = 0;
    const long long replays = cdiv(cfg->d_max, kShardGraphSteps);
    for (long long rp = 0; rp < replays; ++rp) {
      const cudaError_t e = cudaGraphLaunch(gexec, c0->stream);
      if (e != cudaSuccess) return set_err(RBD_ERR_CUDA, std::string("sharded graph launch: ") + cudaGetErrorString(e));
      R[0]->launches += graph_launches;
      CU(cudaMemcpyAsync(&hd[rp & 1], &ptr<DevState>(c0->state)->done, sizeof(int),
                         cudaMemcpyDeviceToHost, c0->stream));
      CU(cudaEventRecord(ev[rp & 1], c0->stream));
      if (rp > 0) {   // the previous replay's flag; this replay is already queued
        CU(cudaEventSynchronize(ev[(rp - 1) & 1]));
        if (hd[(rp - 1) & 1]) break;
      }
    }
  } else {
    for (long long step = 0; step < cfg->d_max; ++step) {
      TRY(enqueue_shard_step(R, ex, sh, m, ldx, d_cap, pay_stride, vec, grids, ranks_id));
      if ((step & 3) == 3 || step + 1 == cfg->d_max) {
        CU(cudaMemcpyAsync((void*)&R[0]->h_state->done, &ptr<DevState>(R[0]->state)->done, sizeof(int),
                           cudaMemcpyDeviceToHost, R[0]->stream));
        CU(cudaStreamSynchronize(R[0]->stream));
        if (R[0]->h_state->done) break;
      }
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
    result->reserved = use_graph ? 1 : 0;   // 1: steps replayed from a CUDA graph
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

int rbd_shard_pick(const double* recs, int nranks, double* best_r, int64_t* best_j, int* owner) {
  if (!recs || nranks < 1) return set_err(RBD_ERR_INVALID_ARGUMENT, "shard_pick: bad records");
  double v;
  long long j;
  const int r = rbdsel::pick(recs, nranks, 2, &v, &j);
  if (best_r) *best_r = v;
  if (best_j) *best_j = r >= 0 ? j : -1;
  if (owner) *owner = r;
  return RBD_OK;
}

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
  return sharded_decompose(R, ex, sh, m, ldx, n_global, cfg, h_selected, h_history, result,
                           std::vector<int>{ctx->rank});
}

int rbd_decompose_sharded_virtual(rbd_ctx_t ctx, int nranks, const double* const* dX_shards,
                                  const int64_t* n_locals, int64_t m, int64_t ldx,
                                  const rbd_config_t* cfg, double* const* dY_ranks,
                                  double* const* dT_ranks, int64_t* h_selected, double* h_history,
                                  rbd_result_t* result) {
  if (!ctx || !cfg || nranks < 1 || nranks > 16)
    return set_err(RBD_ERR_INVALID_ARGUMENT, "virtual sharded: bad arguments (1..16 ranks)");
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
  std::vector<int> ids(nranks);
  for (int r = 0; r < nranks; ++r) ids[r] = r;
  int rc = sharded_decompose(R, ex, sh, m, ldx, off, cfg, h_selected, h_history, result, ids);
  for (auto c : R) ctx->launches += c->launches;
  return rc;
}

}  // extern "C"
