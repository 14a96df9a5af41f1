// rbd_shard.cu — the multi-GPU (column-sharded) greedy loop behind the C ABI
// (SURVEY §8(e)): NCCL payload exchange and virtual ranks.
#include "rbd_capi_internal.h"
#include "rbd_persistent.cuh"

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
