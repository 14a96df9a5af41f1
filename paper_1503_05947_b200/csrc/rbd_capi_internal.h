// rbd_capi_internal.h — shared by the C-ABI translation units (rbd_capi.cu:
// context, decompose drivers, mgs; rbd_ws.cu: the ErrorWorkspace API;
// rbd_project_capi.cu: project / reconstruct / compress / classify;
// rbd_shard.cu: the multi-GPU loop): the context and workspace structs, device
// scratch buffers, error plumbing and the launch helpers the units share. Not
// part of the C ABI.
#pragma once

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
#include "rbd_device.cuh"   // shared types (DevState, Rec, SweepArgs); each unit includes its kernels
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: phase ranges for nsys / ncu --nvtx

using namespace rbdk;

void rbd_comm_release(rbd_ctx_t ctx);

namespace rbdc {


// records msg as the thread's rbd_last_error() (defined in rbd_capi.cu)
inline int set_err(int code, const std::string& msg) {
  return rbd_internal_set_error(code, msg.c_str());
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

// NVTX range over a host-side phase (the reference times its phases
// with steady_clock in tools/main.cpp:31-33,171-177). Free when no tool attaches.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  void end() {
    if (open) nvtxRangePop();
    open = false;
  }
  ~NvtxRange() { end(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
  bool open = true;
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

inline int ensure(DevBuf& b, size_t bytes) {
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

inline void release(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}

template <typename T>
T* ptr(DevBuf& b) {
  return static_cast<T*>(b.p);
}

inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

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

}  // namespace rbdc

using namespace rbdc;


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
  cudaStream_t up_stream = nullptr;    // rbd_decompose_host_many: uploads of the next X
  DevBuf hX2;                          // rbd_decompose_host_many: two device X buffers
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
  DevBuf wd_yslice;                          // persistent weighted loop: YAY-row slice partials
  DevBuf forced;                             // rbd_set_forced_selection (test instrumentation)
  std::vector<long long> forced_h;
  DevBuf nn_part, nn_coords;               // classify: split minima, query coordinates
  DevBuf pj_ws;                            // K5 split-K partial slices
  DevBuf send, recv;                       // sharded mode: payload (-0.0-padded) and its allreduce
  DevBuf srec, rrec;                       // sharded mode: 16-byte records and their allgather
  double* h_done = nullptr;                // sharded mode: pinned done flags of the graph replays
  // host-buffer entries (project/reconstruct/compress/classify/mgs_project/
  // ws_extend _host): device scratch kept between calls instead of a
  // cudaMalloc/cudaFree pair (and the implicit device sync of cudaFree) per call
  DevBuf hs[5];
  // device-resident model entries (rbd_model.cu): two buffers per operand for
  // the pipelined batch stream, plus the D2H stream
  DevBuf pm_X[2], pm_T[2], pm_E[2];
  cudaStream_t d2h_stream = nullptr;
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


namespace rbdc {

// ---- launch helpers defined in rbd_capi.cu, used by the other units ----
int launch_sweep(rbd_ctx_t ctx, const SweepArgs& a, int vec, int mode, bool stream_a,
                 long long ncols_max);
int finalize_grid(rbd_ctx_t ctx, long long n);
long long gemv_grid(long long m);
int enqueue_init(rbd_ctx_t ctx, const double* X, long long m, long long n, long long ldx,
                 double* partial, double* colsq, double* resid, DevState* st);
int diag_vec_grid(rbd_ctx_t ctx, long long m);
size_t persist_smem(long long dcap, bool diag = false, bool fold = false);
long long y_delay(int grid, bool xf32 = false);
int persistent_grid(rbd_ctx_t ctx, int vec, long long d_max, bool diag = false, bool xf32 = false,
                    bool fold = false);
int ensure_loop_buffers(rbd_ctx_t ctx, long long m, long long n, long long d_max);
int validate_after_init(const rbd_config_t* cfg, long long m, long long n, const DevState& hs,
                        bool diag_supplied = false, double diag_max = 0.0);
int start_column(const rbd_config_t* cfg, long long n, long long* out);
double breakdown_tolerance(const rbd_config_t* cfg, long long m, double max_colsq);
int check_diagonal(const double* h, int64_t len);

}  // namespace rbdc
