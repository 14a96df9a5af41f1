/* rbd_cuda.h — C ABI of the B200-native RBD greedy loop (arXiv 1503.05947).
 *
 * This is the drop-in boundary under the reference's C++ API
 * (proj/include/rbd/decompose.hpp:61-77, workspace.hpp:34-54). Every entry
 * point takes plain pointers and sizes; no torch or Eigen types cross it.
 * The C++ mirror of the reference API (include/rbd/<name>.hpp) and the Python
 * package (paper_1503_05947_b200) are thin layers over these functions.
 *
 * Layouts (all fp64):
 *   X      m x n column-major, leading dimension ldx >= m  (reference types.hpp:9-10)
 *   Y      m x cap column-major, leading dimension m          (RbdModel::Y)
 *   T      cap x n ROW-major: T[k*n + j] = row k of the reference's d x n T
 *          (the reference writes T row-major in its model file, io.cpp:563-564)
 * Device pointers are CUDA device addresses on the context's device; host
 * pointers are ordinary (pageable or pinned) host memory.
 *
 * Errors: every function returns an rbd_status (0 = ok). The message of the
 * last failure on the calling thread is returned by rbd_last_error(). Status
 * codes map one-to-one onto the reference's rbd::Error subclasses
 * (proj/include/rbd/errors.hpp:9-77).
 *
 * Threading: one rbd_ctx per host thread; calls on distinct contexts are
 * reentrant. Results are deterministic: the same inputs and config give
 * bit-identical Y, T, selected and history (test_decompose.cpp:128-137),
 * including across 1/2/4/8 column shards (summation order depends on m only).
 */
#ifndef RBD_CUDA_H
#define RBD_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RBD_ABI_VERSION 1

typedef enum {
  RBD_OK = 0,
  RBD_ERR_INVALID_ARGUMENT = 1,   /* rbd::InvalidArgument   errors.hpp:62-65 */
  RBD_ERR_INCOMPATIBLE_WEIGHT = 2,/* rbd::IncompatibleWeight errors.hpp:21-24 */
  RBD_ERR_DEGENERATE_INPUT = 3,   /* rbd::DegenerateInput   errors.hpp:27-30 */
  RBD_ERR_INDEX_OUT_OF_RANGE = 4, /* rbd::IndexOutOfRange   errors.hpp:39-42 */
  RBD_ERR_DIMENSION_MISMATCH = 5, /* rbd::DimensionMismatch errors.hpp:15-18 */
  RBD_ERR_NOT_POSITIVE = 6,       /* rbd::NotPositive       errors.hpp:33-36 */
  RBD_ERR_NO_CONVERGENCE = 7,     /* rbd::NoConvergence     errors.hpp:45-48 */
  RBD_ERR_UNSUPPORTED_FORMAT = 8, /* rbd::UnsupportedFormat errors.hpp:54-57 */
  RBD_ERR_IO = 9,                 /* rbd::IoError           errors.hpp:59-62 */
  RBD_ERR_PARSE = 10,             /* rbd::ParseError        errors.hpp:64-77 ("path:line: what") */
  RBD_ERR_CUDA = 100,             /* CUDA runtime failure (maps to rbd::Error) */
  RBD_ERR_NCCL = 101,             /* NCCL failure (maps to rbd::Error) */
  RBD_ERR_OUT_OF_MEMORY = 102     /* device allocation failure (maps to rbd::Error) */
} rbd_status;

typedef enum { RBD_START_FIXED_COLUMN = 0, RBD_START_SEEDED_RANDOM = 1 } rbd_start_kind;
typedef enum { RBD_WEIGHT_IDENTITY = 0, RBD_WEIGHT_DIAGONAL = 1, RBD_WEIGHT_SPARSE_SPD = 2 } rbd_weight_kind;

/* Mirrors rbd::RbdConfig + rbd::StartSpec (decompose.hpp:14-36). */
typedef struct {
  int64_t d_max;            /* 1 <= d_max <= n, checked at decompose time          */
  double eps_R;             /* absolute stop tolerance on E_cur                    */
  int32_t start_kind;       /* rbd_start_kind (default fixed column)               */
  int32_t reorthogonalize;  /* force the second orthogonalisation pass             */
  int64_t start_column;     /* fixed start column (default 0)                      */
  uint64_t start_seed;      /* seed for RBD_START_SEEDED_RANDOM                    */
  double breakdown_tol;     /* < 0: use eps_R (reference default -1.0)             */
  int32_t weight_kind;      /* rbd_weight_kind; DIAGONAL via rbd_decompose_diag_*  */
  int64_t weight_dim;       /* dimension of a non-identity weight (compat check)   */
} rbd_config_t;

typedef struct rbd_ctx_s* rbd_ctx_t;
typedef struct rbd_ws_s* rbd_ws_t;

/* Result counters of a decomposition (the rest goes to caller buffers). */
typedef struct {
  int64_t d;            /* accepted basis vectors (RbdModel::d)               */
  int32_t breakdown;    /* 1 if the loop ended on an orthogonalisation breakdown */
  int32_t reserved;
  double breakdown_tol; /* effective breakdown tolerance (decompose.cpp:73-74) */
  double max_col_norm;  /* max_j ||x_j|| (noise-floor input, decompose.cpp:70) */
  double init_ms;       /* device time of the K1 init pass (CUDA events)      */
  double loop_ms;       /* device time from the first greedy step to the stop  */
  int64_t launches;     /* kernels launched by this call                       */
} rbd_result_t;

const char* rbd_last_error(void);
int rbd_abi_version(void);
void rbd_config_default(rbd_config_t* cfg);

/* Context: owns the device, a stream, scratch buffers and captured graphs. */
int rbd_ctx_create(int device, rbd_ctx_t* out);
int rbd_ctx_destroy(rbd_ctx_t ctx);
/* Use an external stream (e.g. torch's current stream); NULL = context stream. */
int rbd_ctx_set_stream(rbd_ctx_t ctx, void* cuda_stream);
/* Number of kernel launches issued by this context since creation (evidence). */
int64_t rbd_ctx_launch_count(rbd_ctx_t ctx);

/* Test instrumentation for the parity protocol (no reference
 * counterpart): later decompose calls on ctx start at h_selected[0] and take
 * h_selected[k] instead of the greedy argmax at step k < count (the residual
 * history still records the argmax residual, decompose.cpp:97-99). Used to
 * re-run the B200 loop on the oracle's selection after an admissible near-tie
 * divergence so Y, T and residuals stay comparable for all steps. Implemented
 * on the persistent loop (identity and diagonal weight); other paths return
 * RBD_ERR_INVALID_ARGUMENT. count = 0 clears. */
int rbd_set_forced_selection(rbd_ctx_t ctx, const int64_t* h_selected, int64_t count);
int rbd_ctx_synchronize(rbd_ctx_t ctx);
/* The cudaStream_t the context launches on (for event timing by callers). */
void* rbd_ctx_stream(rbd_ctx_t ctx);

/* rbd::decompose (decompose.cpp:53-111) on device-resident X.
 * dY: m x d_max (ld m), dT: d_max x n row-major, both device buffers.
 * h_selected / h_history: host arrays of length d_max. */
int rbd_decompose_device(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx,
                         const rbd_config_t* cfg, double* dY, double* dT, int64_t* h_selected,
                         double* h_history, rbd_result_t* result);

/* rbd::decompose with HOST buffers: X is uploaded, Y/T downloaded inside the
 * call (the reference-facing, end-to-end entry). hY: m x d_max col-major,
 * hT: d_max x n row-major (rows >= result->d are left untouched). */
int rbd_decompose_host(rbd_ctx_t ctx, const double* hX, int64_t m, int64_t n, int64_t ldx,
                       const rbd_config_t* cfg, double* hY, double* hT, int64_t* h_selected,
                       double* h_history, rbd_result_t* result);

/* fp32 storage mode of rbd::decompose (BASELINE north_star's optional fp32
 * mode; same contract as rbd_decompose_device / _host otherwise): X is held
 * in fp32 (half the HBM bytes the per-step sweep streams), every product and
 * sum is fp64 on the exact value of each element, and Y, T, the residuals and
 * the history are fp64. The result is therefore the fp64 algorithm run on the
 * fp32-valued matrix (parity: the fp64 oracle on X rounded to fp32, to the
 * fp64 tolerances). Identity weight, persistent loop (d_max <= 4096);
 * otherwise RBD_ERR_INVALID_ARGUMENT. */
int rbd_decompose_device_f32(rbd_ctx_t ctx, const float* dX, int64_t m, int64_t n, int64_t ldx,
                             const rbd_config_t* cfg, double* dY, double* dT, int64_t* h_selected,
                             double* h_history, rbd_result_t* result);
int rbd_decompose_host_f32(rbd_ctx_t ctx, const float* hX, int64_t m, int64_t n, int64_t ldx,
                           const rbd_config_t* cfg, double* hY, double* hT, int64_t* h_selected,
                           double* h_history, rbd_result_t* result);

/* rbd::decompose over a sequence of `count` host matrices of one shape and
 * config (the end-to-end entry for a stream of inputs): the H2D upload of
 * matrix i+1 runs on a second stream (copy engine) while matrix i's greedy
 * loop runs, with two device X buffers. Per matrix the outputs and errors are
 * rbd_decompose_host's (hY[i], hT[i], h_selected[i], h_history[i],
 * results[i]; any of the pointer arrays may be NULL). Page-locked X is needed
 * for the overlap. Stops at the first failing matrix and returns its status. */
int rbd_decompose_host_many(rbd_ctx_t ctx, int64_t count, const double* const* hX, int64_t m,
                            int64_t n, int64_t ldx, const rbd_config_t* cfg, double* const* hY,
                            double* const* hT, int64_t* const* h_selected, double* const* h_history,
                            rbd_result_t* results);
int rbd_decompose_host_many_f32(rbd_ctx_t ctx, int64_t count, const float* const* hX, int64_t m,
                                int64_t n, int64_t ldx, const rbd_config_t* cfg, double* const* hY,
                                double* const* hT, int64_t* const* h_selected,
                                double* const* h_history, rbd_result_t* results);

/* rbd::decompose with cfg.weight = WeightSpec::diagonal(diag) (
 * reference decompose.cpp:53-111, weight.cpp:11-21, workspace.cpp:24-29,61-99,
 * 114-122). Y and T are Euclidean as in the reference; the weight steers the
 * greedy selection through the A-norm residual. diag: diag_len positive finite
 * doubles (device memory for _device, host memory for _host); InvalidArgument
 * for an empty/non-positive/non-finite diagonal (weight.cpp:11-17),
 * IncompatibleWeight when diag_len != m (decompose.cpp:61-62). cfg->weight_kind
 * and weight_dim are taken from the call. */
int rbd_decompose_diag_device(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx,
                              const rbd_config_t* cfg, const double* d_diag, int64_t diag_len,
                              double* dY, double* dT, int64_t* h_selected, double* h_history,
                              rbd_result_t* result);
int rbd_decompose_diag_host(rbd_ctx_t ctx, const double* hX, int64_t m, int64_t n, int64_t ldx,
                            const rbd_config_t* cfg, const double* h_diag, int64_t diag_len,
                            double* hY, double* hT, int64_t* h_selected, double* h_history,
                            rbd_result_t* result);

/* rbd::mgs_project (decompose.cpp:12-33) on device vectors: orthonormalise dv
 * against the k orthonormal columns of dB (ld ldb). On success *ok = 1 and
 * dxi/norm hold the unit vector and pre-normalisation norm; *ok = 0 on
 * breakdown (the reference's std::nullopt). */
int rbd_mgs_project(rbd_ctx_t ctx, const double* dv, int64_t m, const double* dB, int64_t k,
                    int64_t ldb, double breakdown_tol, int reorthogonalize, double* dxi,
                    double* norm, int* ok);

/* ErrorWorkspace, identity weight (workspace.hpp:18-54). The workspace keeps
 * a pointer to dX (not owned, workspace.hpp:15-17) and up to cap T rows. */
int rbd_ws_init(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx, int64_t cap,
                rbd_ws_t* out);
int rbd_ws_destroy(rbd_ws_t ws);
int rbd_ws_extend(rbd_ws_t ws, const double* dxi);          /* workspace.cpp:43-60 */
int rbd_ws_scan(rbd_ws_t ws, double* e_cur, int64_t* argmax); /* workspace.cpp:101-125 */
int rbd_ws_error_sq(rbd_ws_t ws, int64_t j, const double* h_c, int64_t clen, double* out); /* :84-99 */
int64_t rbd_ws_d(rbd_ws_t ws);
int rbd_ws_read(rbd_ws_t ws, double* h_col_sq, double* h_residual_sq, double* h_yax /* d x n row-major */);

/* Host-buffer variants used by the C++ mirror (include/rbd/<name>.hpp). */
int rbd_mgs_project_host(rbd_ctx_t ctx, const double* hv, int64_t m, const double* hB, int64_t k,
                         int64_t ldb, double breakdown_tol, int reorthogonalize, double* hxi,
                         double* norm, int* ok);
/* Workspace over a device copy of host X (owned by the workspace). */
/* ErrorWorkspace with a diagonal weight (workspace.cpp:24-29 init, 61-79 extend:
 * the yax row X'(a o xi) and the Y'AY row; 84-99 error_sq with Y'AY). The
 * residual_sq kept by the identity workspace is not maintained for a weight
 * (as in the reference): scan with rbd_ws_scan_T. d_diag: diag_len device
 * doubles (host doubles for _host); InvalidArgument for a bad diagonal,
 * IncompatibleWeight when diag_len != m. */
int rbd_ws_init_diag(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx,
                     int64_t cap, const double* d_diag, int64_t diag_len, rbd_ws_t* out);
int rbd_ws_init_diag_host(rbd_ctx_t ctx, const double* hX, int64_t m, int64_t n, int64_t ldx,
                          int64_t cap, const double* h_diag, int64_t diag_len, rbd_ws_t* out);
/* residual_scan(ws, T) for any weight (workspace.cpp:101-125): error_sq of every
 * column with c = T[:, j], T the d x n coefficients row-major (device / host). */
int rbd_ws_scan_T(rbd_ws_t ws, const double* dT, double* e_cur, int64_t* argmax);
int rbd_ws_scan_T_host(rbd_ws_t ws, const double* hT, double* e_cur, int64_t* argmax);
/* Y'AY (d x d row-major) of a diagonal workspace. */
int rbd_ws_read_yay(rbd_ws_t ws, double* h_yay);
int rbd_ws_init_host(rbd_ctx_t ctx, const double* hX, int64_t m, int64_t n, int64_t ldx,
                     int64_t cap, rbd_ws_t* out);
int rbd_ws_extend_host(rbd_ws_t ws, const double* hxi);

/* Out-of-sample compression (decompose.cpp:113-117, batched) plus the
 * identity error indicator err_j = max(||x_j||^2 - ||t_j||^2, 0) (Eq. 3,
 * workspace.cpp:88-97). dY m x d (ld ldy), dXn m x N (ld ldx);
 * dTn d x N column-major (ld d), d_err length N (may be NULL). */
int rbd_project_batch(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                      const double* dXn, int64_t N, int64_t ldx, double* dTn, double* d_err);
/* fp32 mode of the out-of-sample compression (BASELINE north_star, 1e-4
 * parity): Y and X_new in fp32, T_new = Y'X_new on the tcgen05 tensor cores
 * (kind::tf32, 3xTF32 split, TMEM accumulators, TMA operand staging); the
 * error indicator is accumulated in fp64. dTn: d x N column-major fp32.
 * ldy/ldx must be multiples of 4 and the bases 16-byte aligned (TMA). */
int rbd_project_batch_f32(rbd_ctx_t ctx, const float* dY, int64_t m, int64_t d, int64_t ldy,
                          const float* dXn, int64_t N, int64_t ldx, float* dTn, double* d_err);
/* rbd::reconstruct (decompose.cpp:119-123): dv = Y c (dc length d). */
int rbd_reconstruct(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                    const double* dc, double* dv);
/* compress_matrix (decompose.cpp:125) on device: V (m x n, column-major, ld ldv)
 * = Y (m x d, ld ldy) T, with T the d x n decompose T in the library's
 * row-major layout (T[k*ldt + j]); FP64 tensor cores (DMMA). */
int rbd_compress_device(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                        const double* dT, int64_t n, int64_t ldt, double* dV, int64_t ldv);
/* rbd::compress_matrix (decompose.cpp:125): V = Y C, C d x N column-major
 * (ld d), V m x N column-major (ld m). */
int rbd_reconstruct_batch(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                          const double* dC, int64_t N, double* dV);
int rbd_compress_host(rbd_ctx_t ctx, const double* hY, int64_t m, int64_t d, const double* hC,
                      int64_t N, double* hV);
/* Host-buffer variants (upload, kernel, download inside the call). */
int rbd_project_host(rbd_ctx_t ctx, const double* hY, int64_t m, int64_t d, const double* hXn,
                     int64_t N, double* hTn, double* h_err);
int rbd_reconstruct_host(rbd_ctx_t ctx, const double* hY, int64_t m, int64_t d,
                         const double* hc, double* hv);

/* ---- Device-resident model (SURVEY §8(b) rbd_model_t) ----
 * An RbdModel (decompose.hpp:39-46) whose Y (m x d, column-major, ld m) and T
 * (d x n, row-major) live in HBM, so the reference's per-vector callers
 * (project: classify.cpp:22-23, tools/main.cpp:149-158; reconstruct:
 * main.cpp:128-145) pay no Y upload or allocation per call. Created from host
 * or device buffers (copied), or read from an RBD1 file straight into HBM
 * (read_model, io.cpp:574-622). Usable from any context on the same device;
 * immutable after creation. */
typedef struct rbd_model_s* rbd_model_t;
/* Y: m x d (ld ldy >= m), T: d x n row-major (ld n); y_on_device selects
 * whether Y and T are device (1) or host (0) pointers. T may be NULL (a model
 * for project / reconstruct only); history (host, length d) may be NULL. */
int rbd_model_create(rbd_ctx_t ctx, int64_t m, int64_t n, int64_t d, const double* Y, int64_t ldy,
                     const double* T, int y_on_device, const double* h_history, double eps_r,
                     rbd_model_t* out);
/* read_model into a device-resident model (diagonal weights are validated as
 * WeightSpec::diagonal; tag 2 models load with weight_kind 2 and no values). */
int rbd_model_load(rbd_ctx_t ctx, const char* path, rbd_model_t* out);
int rbd_model_free(rbd_model_t model);
/* Shape, device pointers (Y ld m; T row-major), eps_R, weight kind. */
int rbd_model_info(rbd_model_t model, int64_t* m, int64_t* n, int64_t* d, const double** dY,
                   const double** dT, double* eps_r, int* weight_kind);
/* Host copies of history[d] and (weight kind 1) diag[m]; either may be NULL. */
int rbd_model_read_vectors(rbd_model_t model, double* h_history, double* h_diag);
/* project (decompose.cpp:113-117), batched, HOST buffers: T_new = Y'X_new
 * (d x N column-major, ld d) and err_j = max(||x_j||^2 - ||t_j||^2, 0) (Eq. 3;
 * h_err may be NULL). X_new: m x N (ld ldx >= m). The upload goes into
 * context-owned device scratch that is kept between calls. */
int rbd_project_model(rbd_ctx_t ctx, rbd_model_t model, const double* hXn, int64_t N, int64_t ldx,
                      double* hTn, double* h_err);
/* reconstruct (decompose.cpp:119-123), batched, HOST buffers: V = Y C, C d x N
 * column-major (ld d), V m x N column-major (ld m). */
int rbd_reconstruct_model(rbd_ctx_t ctx, rbd_model_t model, const double* hC, int64_t N, double* hV);
/* A stream of `count` out-of-sample batches of N columns each (BASELINE
 * config 4: 16 batches of 16,384): the H2D of batch i+1 runs on a copy stream
 * while batch i is contracted (K5, DMMA) and batch i-1's T_new/err come back
 * on a third stream; two device buffers per operand. Page-locked inputs and
 * outputs are needed for the overlap. Same bits as rbd_project_model per
 * batch. h_err[i] may be NULL (or h_err itself). */
int rbd_project_host_many(rbd_ctx_t ctx, rbd_model_t model, int64_t count,
                          const double* const* hXn, int64_t N, int64_t ldx, double* const* hTn,
                          double* const* h_err);
/* fp32 mode of the same stream (north star: fp32 Y and X_new, 1e-4 parity):
 * K6 (tcgen05 kind::tf32, 3xTF32) on an fp32 copy of Y the model keeps;
 * T_new fp32, err accumulated in fp64. */
int rbd_project_host_many_f32(rbd_ctx_t ctx, rbd_model_t model, int64_t count,
                              const float* const* hXn, int64_t N, int64_t ldx, float* const* hTn,
                              double* const* h_err);

/* Measurement hook: run the fused sweep kernel (K2) `reps` times back to back
 * on dX with vector dy and return the mean device time per launch (CUDA
 * events on the context stream). Used by bench.py for the roofline figure. */
int rbd_time_sweep(rbd_ctx_t ctx, const double* dX, int64_t m, int64_t n, int64_t ldx,
                   const double* dy, int reps, double* ms_per_launch);

/* ---- multi-GPU (one process per GPU; X sharded by contiguous column blocks,
 *      Y replicated) ---- */
#define RBD_UNIQUE_ID_BYTES 128
/* The winner rule of the per-step record exchange (host-callable; the device
 * kernels run the same code, csrc/rbd_select.h): recs[2r] = rank r's best
 * residual, recs[2r+1] = its GLOBAL column index as int64 bits (-1: none).
 * Largest residual, ties to the smallest global index (the reference's strict
 * '>' scan, workspace.cpp:107-113). *owner = -1 when no rank has a candidate. */
int rbd_shard_pick(const double* recs, int nranks, double* best_r, int64_t* best_j, int* owner);
int rbd_comm_unique_id(char out[RBD_UNIQUE_ID_BYTES]);
int rbd_ctx_init_comm(rbd_ctx_t ctx, int rank, int world, const char id[RBD_UNIQUE_ID_BYTES]);
/* Sharded decompose: this rank owns global columns [col_offset, col_offset+n_local)
 * of an m x n_global X. dT_local: d_max x n_local row-major. selected holds
 * GLOBAL column indices; Y/selected/history are identical on every rank. Per
 * step: the local fused sweep, an ncclAllGather of 16-byte records, the
 * owner's payload {col_sq, x_j, T[0:k+1, j]} by a -0.0-padded ncclAllReduce
 * (exact), replayed from a CUDA graph of 8 steps (RBD_SHARD_GRAPH=0: eager;
 * result->reserved = 1 when the graph ran). */
int rbd_decompose_sharded(rbd_ctx_t ctx, const double* dX_local, int64_t m, int64_t n_local,
                          int64_t ldx, int64_t col_offset, int64_t n_global,
                          const rbd_config_t* cfg, double* dY, double* dT_local,
                          int64_t* h_selected, double* h_history, rbd_result_t* result);

/* Single-device emulation of the sharded loop: nranks column shards (shard r
 * holds n_locals[r] consecutive global columns) stepped in lockstep in this
 * process, with the payload allgather done by device copies. Same kernels and
 * protocol as rbd_decompose_sharded; used to test cross-shard bitwise identity
 * on one GPU. dY_ranks[r]: m x d_max per rank (replicated Y); dT_ranks[r]:
 * d_max x n_locals[r] row-major. */
int rbd_decompose_sharded_virtual(rbd_ctx_t ctx, int nranks, const double* const* dX_shards,
                                  const int64_t* n_locals, int64_t m, int64_t ldx,
                                  const rbd_config_t* cfg, double* const* dY_ranks,
                                  double* const* dT_ranks, int64_t* h_selected, double* h_history,
                                  rbd_result_t* result);

/* ---- Batched Classifier::predict (classify.cpp:22-34) ----
 * For every query column v_q of dQ (m x Q, ld ldq): c_q = Y'v_q (K5), then the
 * training column j minimising ||T[:,j] - c_q||^2 (difference form, summed in
 * coordinate order; smallest j on ties, classify.cpp:24-32). dT is the d x
 * n_train decompose T, row-major (T[k*n_train + j]). d_best[Q] (int64) and
 * optional d_dist[Q] are device outputs; the label lookup stays with the caller
 * (Classifier::labels). */
int rbd_classify_batch(rbd_ctx_t ctx, const double* dY, int64_t m, int64_t d, int64_t ldy,
                       const double* dT, int64_t n_train, const double* dQ, int64_t Q,
                       int64_t ldq, int64_t* d_best, double* d_dist);
/* Same with host buffers (Y m x d col-major ld m, T row-major, Q m x Q ld m). */
int rbd_classify_host(rbd_ctx_t ctx, const double* hY, int64_t m, int64_t d, const double* hT,
                      int64_t n_train, const double* hQ, int64_t Q, int64_t* h_best,
                      double* h_dist);
/* The nearest-column step alone, for query coordinates dC (d x Q, ld ldc). */
int rbd_nearest_columns(rbd_ctx_t ctx, const double* dC, int64_t d, int64_t Q, int64_t ldc,
                        const double* dT, int64_t n_train, int64_t* d_best, double* d_dist);

/* ---- RBD1 model container (io.cpp:527-622, io.hpp:51-64) ----
 * Layout (little-endian): "RBD1" | u64 m, n, d | u8 weight tag | f64 Y (m x d,
 * column-major) | f64 T (d x n, row-major) | f64 eps_R | f64 history[d] |
 * (tag 1) f64 diag[m]; 29-byte header. Y and T may be device or host pointers
 * (device data streams through pinned double buffers on the context stream;
 * ctx may be NULL for host-only use). history (and diag on write) are host
 * arrays; diag may also be device memory. Writes are atomic (path + ".tmp",
 * then rename, io.cpp:60-73). Errors: IoError (cannot open / write / rename),
 * ParseError "path:0: what" (bad magic, implausible dimensions, unknown tag,
 * size mismatch, truncation), DimensionMismatch for inconsistent shapes. */
int rbd_model_write(rbd_ctx_t ctx, const char* path, int64_t m, int64_t n, int64_t d,
                    const double* Y, int64_t ldy, const double* T, double eps_r,
                    const double* h_history, int weight_kind, const double* h_diag);
/* Validates the header and the file size (io.cpp:577-596) and returns the shape. */
int rbd_model_read_header(const char* path, int64_t* m, int64_t* n, int64_t* d, int* weight_kind);
/* Reads a validated file into Y (ld ldy >= m), T (d x n row-major), eps_r,
 * h_history[d] and (tag 1) h_diag[m]. */
int rbd_model_read(rbd_ctx_t ctx, const char* path, double* Y, int64_t ldy, double* T,
                   double* eps_r, double* h_history, double* h_diag);

#ifdef __cplusplus
}
#endif
#endif /* RBD_CUDA_H */
