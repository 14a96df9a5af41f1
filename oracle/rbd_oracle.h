/* TEST INFRASTRUCTURE ONLY — NOT PART OF THE PRODUCT.
 *
 * CPU restatement ("oracle") of the reference RBD greedy loop (identity and
 * diagonal weights), written with plain loops (no Eigen: Eigen 3.4 is absent from this image,
 * so /root/reference cannot be compiled — see DESIGN.md §Oracle).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library, and only as the checker or the
 * timed CPU baseline. The product path (paper_1503_05947_b200) never links it.
 *
 * Parity pinning: the restatement is validated against every known-answer value
 * and property test the reference holds for this path (tests/test_oracle_*.py:
 * SPEC.md:67-71,201-204 examples, test_decompose.cpp:29-289,
 * test_workspace.cpp:28-212 (identity), acceptance.cpp:95-297 criteria 1-4 with
 * the recorded values of proj/test_output.txt:9-15, test_smoke.py:7-28).
 * The fixture generators below reproduce the reference test helpers bit for bit
 * (same libstdc++ std::mt19937_64 / std::normal_distribution draws).
 *
 * Status codes mirror include/rbd_cuda.h (and rbd::Error subclasses,
 * proj/include/rbd/errors.hpp:9-77).
 */
#ifndef RBD_ORACLE_H
#define RBD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_INVALID_ARGUMENT = 1,
  ORC_INCOMPATIBLE_WEIGHT = 2,
  ORC_DEGENERATE_INPUT = 3,
  ORC_INDEX_OUT_OF_RANGE = 4,
  ORC_DIMENSION_MISMATCH = 5
};

const char* orc_last_error(void);

/* rbd::decompose (proj/src/decompose.cpp:53-111), identity weight.
 * X: m x n column-major, leading dimension ldx >= m.
 * Outputs (capacity d_max): Y m x d_max column-major (ld m); T d_max x n
 * ROW-major (T[k*n + j] = row k of the reference's d x n T); selected; history.
 * nthreads: OpenMP threads for the two per-step X passes (1 = the reference's
 * single thread). Results are bitwise independent of nthreads. */
int orc_decompose(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t d_max,
                  double eps_R, int start_kind, int64_t start_column, uint64_t start_seed,
                  int reorthogonalize, double breakdown_tol, int nthreads, double* Y,
                  double* T, int64_t* selected, double* history, int64_t* d_out);

/* Same loop, stopping after at most max_steps accepted vectors (bounded CPU
 * baseline sample); identical arithmetic. */
int orc_decompose_steps(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t d_max,
                        double eps_R, int start_kind, int64_t start_column,
                        uint64_t start_seed, int reorthogonalize, double breakdown_tol,
                        int nthreads, int64_t max_steps, double* Y, double* T,
                        int64_t* selected, double* history, int64_t* d_out);

/* Same loop with the options the config-scale parity tests and the CPU
 * baseline need: x_passes = 2 is the reference's two X passes per step
 * (decompose.cpp:93 and workspace.cpp:51); 1 reuses the first pass's values
 * (identical bits, half the CPU time). t_init_s / t_loop_s (may be NULL): wall
 * time of validation + workspace_init and of the greedy loop. */
int orc_decompose_ex(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t d_max,
                     double eps_R, int start_kind, int64_t start_column, uint64_t start_seed,
                     int reorthogonalize, double breakdown_tol, int nthreads, int64_t max_steps,
                     int x_passes, double* Y, double* T, int64_t* selected, double* history,
                     int64_t* d_out, double* t_init_s, double* t_loop_s);

/* Column-block pieces of the same loop (for X streamed in blocks):
 * sq[j] = ||x_j||^2 (dot8 order) with the allFinite / all-zero flags, and
 * row[j] = xi . x_j. */
void orc_column_pass(const double* X, int64_t m, int64_t n, int64_t ldx, int nthreads, double* sq,
                     int* all_finite, int* all_zero);
void orc_gemv_t(const double* X, int64_t m, int64_t n, int64_t ldx, const double* xi, double* row,
                int nthreads);

/* rbd::decompose with WeightSpec::diagonal(diag) (decompose.cpp:53-111,
 * weight.cpp:11-21, workspace.cpp:24-29,61-99,114-122). Single-threaded;
 * Y/T/selected/history as orc_decompose. */
int orc_decompose_diag(const double* X, int64_t m, int64_t n, int64_t ldx, const double* diag,
                       int64_t diag_len, int64_t d_max, double eps_R, int start_kind,
                       int64_t start_column, uint64_t start_seed, int reorthogonalize,
                       double breakdown_tol, int64_t max_steps, double* Y, double* T,
                       int64_t* selected, double* history, int64_t* d_out);

/* rbd::mgs_project (decompose.cpp:12-33). Returns 1 with xi/norm filled, 0 on
 * breakdown (std::nullopt), negative on DimensionMismatch. */
int orc_mgs_project(const double* v, int64_t m, const double* basis, int64_t k, int64_t ldb,
                    double breakdown_tol, int reorthogonalize, double* xi, double* norm);

/* ErrorWorkspace identity path (workspace.cpp:9-60, 84-125) and diagonal path
 * (workspace.cpp:24-29, 61-79, 84-99, 114-122). */
typedef struct orc_ws_s* orc_ws_t;
orc_ws_t orc_ws_init(const double* X, int64_t m, int64_t n, int64_t ldx);
/* NULL (ORC_INCOMPATIBLE_WEIGHT in orc_last_error) when diag_len != m. */
orc_ws_t orc_ws_init_diag(const double* X, int64_t m, int64_t n, int64_t ldx, const double* diag,
                          int64_t diag_len);
/* residual_scan with T (row-major d x n), any weight (workspace.cpp:101-125). */
int orc_ws_scan_T(orc_ws_t ws, const double* T, double* e_cur, int64_t* argmax);
/* Y'AY (row-major d x d), diagonal workspaces only. */
int orc_ws_yay(orc_ws_t ws, double* out);
void orc_ws_free(orc_ws_t ws);
int orc_ws_extend(orc_ws_t ws, const double* xi);
int64_t orc_ws_d(orc_ws_t ws);
void orc_ws_col_sq(orc_ws_t ws, double* out);
void orc_ws_residual(orc_ws_t ws, double* out);
void orc_ws_yax_row(orc_ws_t ws, int64_t k, double* out);
int orc_ws_error_sq(orc_ws_t ws, int64_t j, const double* c, int64_t clen, double* out);
int orc_ws_scan(orc_ws_t ws, double* e_cur, int64_t* argmax);

/* project / reconstruct / compress_matrix (decompose.cpp:113-125). */
void orc_project(const double* Y, int64_t m, int64_t d, const double* v, double* c);
void orc_reconstruct(const double* Y, int64_t m, int64_t d, const double* c, double* v);
void orc_project_batch(const double* Y, int64_t m, int64_t d, const double* Xn, int64_t N,
                       int64_t ldx, int nthreads, double* Tn, double* err);

/* Batched Classifier::predict (classify.cpp:22-34): Y m x d (ld m), T d x n_tr
 * row-major, queries m x nq (ld m); best column and its squared distance. */
void orc_predict_batch(const double* Y, int64_t m, int64_t d, const double* T, int64_t n_tr,
                       const double* Qm, int64_t nq, int nthreads, int64_t* best_out,
                       double* dist_out);
/* gen_labeled_blobs (datasets.cpp:67-97), bit-identical draws. */
int orc_gen_labeled_blobs(int n_classes, int per_class, int dim, double spread, uint64_t seed,
                          double* samples, int* labels);

/* Fixture generators restating the reference's test helpers. */
void orc_random_matrix(int64_t m, int64_t n, uint64_t seed, double* out);      /* helpers.hpp:14-21 */
void orc_random_positive(int64_t n, uint64_t seed, double* out);        /* helpers.hpp:28-34 */
void orc_random_low_rank(int64_t m, int64_t n, int64_t r, uint64_t seed, double* out); /* :23-26 */
int orc_gen_grid_matrix(int fid, int64_t n_points, double* out); /* datasets.cpp:30-65 */
int64_t orc_acceptance3_count(void);  /* acceptance.cpp:185-231 column-evaluation count */
int64_t orc_seeded_start(uint64_t seed, int64_t n); /* decompose.cpp:43-46 */

#ifdef __cplusplus
}
#endif
#endif
