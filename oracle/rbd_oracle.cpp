// TEST INFRASTRUCTURE ONLY — NOT PART OF THE PRODUCT (see rbd_oracle.h).
//
// Statement-by-statement CPU restatement of the reference identity-weight RBD
// path with plain loops. Each function cites the reference lines it follows.
// Differences from the reference are limited to floating-point summation order
// inside dot products (Eigen's SIMD partial sums are not reproducible outside
// Eigen; here every dot product uses the fixed 8-way blocked order of dot8()).
#include "rbd_oracle.h"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <ctime>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;

int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}

// Fixed-order dot product: 8 interleaved partial sums (Eigen-like packet
// accumulation, vectorisable without -ffast-math), combined pairwise.
inline double dot8(const double* a, const double* b, int64_t m) {
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t i = 0;
  for (; i + 8 <= m; i += 8)
    for (int k = 0; k < 8; ++k) s[k] += a[i + k] * b[i + k];
  double tail = 0.0;
  for (; i < m; ++i) tail += a[i] * b[i];
  return (((s[0] + s[4]) + (s[1] + s[5])) + ((s[2] + s[6]) + (s[3] + s[7]))) + tail;
}

inline double sqnorm(const double* a, int64_t m) { return dot8(a, a, m); }

inline void axpy(double alpha, const double* x, double* y, int64_t m) {
  for (int64_t i = 0; i < m; ++i) y[i] += alpha * x[i];
}

// row[j] = xi . X(:,j) for all j — the GEMV at decompose.cpp:93 and
// workspace.cpp:51 (computed twice per step by the reference).
void gemv_t(const double* X, int64_t m, int64_t n, int64_t ldx, const double* xi, double* row,
            int nthreads) {
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads) schedule(static) if (nthreads > 1)
#endif
  for (int64_t j = 0; j < n; ++j) row[j] = dot8(xi, X + j * ldx, m);
  (void)nthreads;
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

// mgs_project — decompose.cpp:12-33.
int orc_mgs_project(const double* v, int64_t m, const double* basis, int64_t k, int64_t ldb,
                    double breakdown_tol, int reorthogonalize, double* xi, double* norm_out) {
  std::vector<double> w(v, v + m);                       // :17
  const double entry_norm = std::sqrt(sqnorm(w.data(), m));  // :18
  auto sweep = [&] {                                     // :19-23 (MGS: updated w)
    for (int64_t j = 0; j < k; ++j) {
      const double* bj = basis + j * ldb;
      axpy(-dot8(w.data(), bj, m), bj, w.data(), m);
    }
  };
  sweep();                                               // :24
  if (reorthogonalize || std::sqrt(sqnorm(w.data(), m)) < 0.5 * entry_norm) sweep();  // :28
  const double norm = std::sqrt(sqnorm(w.data(), m));    // :29
  if (norm < breakdown_tol || norm == 0.0) return 0;     // :30 (nullopt)
  for (int64_t i = 0; i < m; ++i) xi[i] = w[i] / norm;   // :31
  *norm_out = norm;                                      // :32
  return 1;
}

int64_t orc_seeded_start(uint64_t seed, int64_t n) {
  // decompose.cpp:43-46 — Eigen::Index is std::ptrdiff_t (long on LP64).
  std::mt19937_64 rng(seed);
  return static_cast<int64_t>(std::uniform_int_distribution<long>(0, static_cast<long>(n) - 1)(rng));
}

// Column pass shared by validation and workspace_init: sq[j] = ||x_j||^2 in
// dot8 order (the value decompose.cpp:70 takes the root of and
// workspace.cpp:22 stores), plus the allFinite (decompose.cpp:57) and
// all-zero (:63-64) flags. Per-column results do not depend on nthreads.
static void column_pass(const double* X, int64_t m, int64_t n, int64_t ldx, int nthreads,
                        double* sq, int* all_finite, int* all_zero) {
  int fin = 1, zero = 1;
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads) schedule(static) reduction(&& : fin, zero) if (nthreads > 1)
#endif
  for (int64_t j = 0; j < n; ++j) {
    const double* x = X + j * ldx;
    bool f = true, z = true;
    for (int64_t i = 0; i < m; ++i) {
      f = f && std::isfinite(x[i]);
      z = z && x[i] == 0.0;
    }
    fin = fin && f;
    zero = zero && z;
    sq[j] = sqnorm(x, m);
  }
  *all_finite = fin;
  *all_zero = zero;
  (void)nthreads;
}

static double now_s() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<double>(ts.tv_sec) + 1e-9 * static_cast<double>(ts.tv_nsec);
}

int orc_decompose_ex(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t d_max,
                     double eps_R, int start_kind, int64_t start_column, uint64_t start_seed,
                     int reorthogonalize, double cfg_breakdown_tol, int nthreads,
                     int64_t max_steps, int x_passes, double* Y, double* T, int64_t* selected,
                     double* history, int64_t* d_out, double* t_init_s, double* t_loop_s) {
  const double t0 = now_s();
  // ---- validation, decompose.cpp:56-64 (same order; the column flags are
  //      computed in one pass and reported in the reference's order) ----
  if (m < 1 || n < 1) return fail(ORC_INVALID_ARGUMENT, "decompose: matrix must be non-empty");
  std::vector<double> sq(n);
  int all_finite = 1, all_zero = 1;
  column_pass(X, m, n, ldx, nthreads, sq.data(), &all_finite, &all_zero);
  if (!all_finite) return fail(ORC_INVALID_ARGUMENT, "decompose: matrix has non-finite entries");
  if (d_max < 1 || d_max > n)
    return fail(ORC_INVALID_ARGUMENT, "decompose: d_max must satisfy 1 <= d_max <= n");
  if (!(eps_R >= 0.0)) return fail(ORC_INVALID_ARGUMENT, "decompose: eps_R must be >= 0");
  // identity weight is always compatible (weight.cpp:71-74)
  if (all_zero) return fail(ORC_DEGENERATE_INPUT, "decompose: zero matrix, no basis can be built");

  // ---- noise floor / breakdown tolerance, decompose.cpp:70-74 ----
  double max_col_norm = 0.0;
  for (int64_t j = 0; j < n; ++j) max_col_norm = std::max(max_col_norm, std::sqrt(sq[j]));
  const double noise_floor =
      max_col_norm * std::sqrt(static_cast<double>(m)) * std::numeric_limits<double>::epsilon() * 16.0;
  const double breakdown_tol =
      std::max(cfg_breakdown_tol < 0.0 ? eps_R : cfg_breakdown_tol, noise_floor);

  // ---- workspace_init (identity), workspace.cpp:21-23,36-40 ----
  std::vector<double> col_sq(n), residual_sq(n);
  for (int64_t j = 0; j < n; ++j) {
    col_sq[j] = std::max(sq[j], 0.0);
    residual_sq[j] = col_sq[j];
  }

  // ---- initial_column, decompose.cpp:37-49 ----
  int64_t i;
  if (start_kind == 0) {
    if (start_column < 0 || start_column >= n)
      return fail(ORC_INDEX_OUT_OF_RANGE, "start column index out of range");
    i = start_column;
  } else {
    i = orc_seeded_start(start_seed, n);
  }
  const double t1 = now_s();

  int64_t d = 0;
  double e_cur = std::numeric_limits<double>::infinity();
  std::vector<double> xi(m), row(n), row2(n);
  while (d < d_max && e_cur > eps_R && d < max_steps) {  // :87
    double nrm;
    // :88-89 (basis = Y.leftCols(d), ld m)
    if (!orc_mgs_project(X + i * ldx, m, Y, d, m, breakdown_tol, reorthogonalize, xi.data(), &nrm))
      break;                                              // :90
    std::memcpy(Y + d * m, xi.data(), sizeof(double) * m);  // :92
    gemv_t(X, m, n, ldx, xi.data(), row.data(), nthreads);  // :93 T.row(d) = xi' X
    std::memcpy(T + d * n, row.data(), sizeof(double) * n);
    selected[d] = i;                                      // :94
    // workspace_extend identity, workspace.cpp:50-53: the reference's second X
    // pass (x_passes == 2). It recomputes the same values with the same
    // summation order, so x_passes == 1 (parity tests at config scale) reuses
    // `row` and gives identical bits at half the CPU time.
    const double* r2 = row.data();
    if (x_passes != 1) {
      gemv_t(X, m, n, ldx, xi.data(), row2.data(), nthreads);
      r2 = row2.data();
    }
    for (int64_t j = 0; j < n; ++j) {
      residual_sq[j] -= r2[j] * r2[j];
      residual_sq[j] = std::max(residual_sq[j], 0.0);
    }
    ++d;                                                  // :96
    // residual_scan identity, workspace.cpp:107-113,123
    double best = -1.0;
    int64_t arg = 0;
    for (int64_t j = 0; j < n; ++j)
      if (residual_sq[j] > best) {
        best = residual_sq[j];
        arg = j;
      }
    e_cur = std::sqrt(best > 0.0 ? best : 0.0);
    history[d - 1] = e_cur;                               // :99
    i = arg;                                              // :101
  }
  if (t_init_s) *t_init_s = t1 - t0;
  if (t_loop_s) *t_loop_s = now_s() - t1;
  if (d == 0)
    return fail(ORC_DEGENERATE_INPUT, "decompose: start column is numerically zero, no basis built");
  *d_out = d;
  return ORC_OK;
}

int orc_decompose_steps(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t d_max,
                        double eps_R, int start_kind, int64_t start_column,
                        uint64_t start_seed, int reorthogonalize, double cfg_breakdown_tol,
                        int nthreads, int64_t max_steps, double* Y, double* T,
                        int64_t* selected, double* history, int64_t* d_out) {
  return orc_decompose_ex(X, m, n, ldx, d_max, eps_R, start_kind, start_column, start_seed,
                          reorthogonalize, cfg_breakdown_tol, nthreads, max_steps, 2, Y, T,
                          selected, history, d_out, nullptr, nullptr);
}

// Pieces of the same loop for a caller that streams X in column blocks (the
// config-3 parity test: 128 GiB of X never sits in host memory at once). The
// caller restates decompose.cpp:53-111 around them; every value is the one the
// whole-matrix loop computes (per-column sums only, same dot8 order).
void orc_column_pass(const double* X, int64_t m, int64_t n, int64_t ldx, int nthreads, double* sq,
                     int* all_finite, int* all_zero) {
  column_pass(X, m, n, ldx, nthreads, sq, all_finite, all_zero);
}
void orc_gemv_t(const double* X, int64_t m, int64_t n, int64_t ldx, const double* xi, double* row,
                int nthreads) {
  gemv_t(X, m, n, ldx, xi, row, nthreads);
}

int orc_decompose(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t d_max,
                  double eps_R, int start_kind, int64_t start_column, uint64_t start_seed,
                  int reorthogonalize, double breakdown_tol, int nthreads, double* Y,
                  double* T, int64_t* selected, double* history, int64_t* d_out) {
  return orc_decompose_steps(X, m, n, ldx, d_max, eps_R, start_kind, start_column, start_seed,
                             reorthogonalize, breakdown_tol, nthreads, INT64_MAX, Y, T,
                             selected, history, d_out);
}

// ---- ErrorWorkspace: identity and diagonal paths ----
struct orc_ws_s {
  const double* X;
  int64_t m, n, ldx, d;
  std::vector<double> col_sq, residual_sq;
  std::vector<std::vector<double>> yax_rows;
  // diagonal weight (workspace.hpp:18-30): diag, yay = Y'AY (row-major d x d,
  // grown per step), a_basis = A*Y (column k = A xi_k)
  std::vector<double> diag;
  std::vector<std::vector<double>> yay;
  std::vector<std::vector<double>> a_basis;
};

orc_ws_t orc_ws_init(const double* X, int64_t m, int64_t n, int64_t ldx) {
  auto* ws = new orc_ws_s{X, m, n, ldx, 0, {}, {}, {}, {}, {}, {}};
  ws->col_sq.resize(n);
  for (int64_t j = 0; j < n; ++j) ws->col_sq[j] = std::max(sqnorm(X + j * ldx, m), 0.0);  // :22,37
  ws->residual_sq = ws->col_sq;                                                           // :38
  return ws;
}

orc_ws_t orc_ws_init_diag(const double* X, int64_t m, int64_t n, int64_t ldx, const double* diag,
                          int64_t diag_len) {
  if (diag_len != m) {  // workspace.cpp:12-13 (compatible_with, weight.cpp:71-74)
    fail(ORC_INCOMPATIBLE_WEIGHT, "weight dimension does not match matrix rows");
    return nullptr;
  }
  auto* ws = new orc_ws_s{X, m, n, ldx, 0, {}, {}, {}, {}, {}, {}};
  ws->diag.assign(diag, diag + m);
  ws->col_sq.resize(n);
  for (int64_t j = 0; j < n; ++j) {  // workspace.cpp:24-29: sum_i x_ij^2 a_i, clamp :37
    const double* x = X + j * ldx;
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += (x[i] * x[i]) * diag[i];
    ws->col_sq[j] = std::max(s, 0.0);
  }
  ws->residual_sq = ws->col_sq;  // :38
  return ws;
}
void orc_ws_free(orc_ws_t ws) { delete ws; }

int orc_ws_extend(orc_ws_t ws, const double* xi) {
  if (ws->diag.empty()) {  // identity, workspace.cpp:50-60
    std::vector<double> row(ws->n);
    gemv_t(ws->X, ws->m, ws->n, ws->ldx, xi, row.data(), 1);
    for (int64_t j = 0; j < ws->n; ++j) {
      ws->residual_sq[j] -= row[j] * row[j];
      ws->residual_sq[j] = std::max(ws->residual_sq[j], 0.0);
    }
    ws->yax_rows.push_back(std::move(row));
    ws->d += 1;
    return ORC_OK;
  }
  // diagonal, workspace.cpp:61-79
  const int64_t m = ws->m, d = ws->d;
  std::vector<double> axi(m);
  for (int64_t i = 0; i < m; ++i) axi[i] = ws->diag[i] * xi[i];  // :64 apply (weight.cpp:83)
  std::vector<double> row(ws->n);
  gemv_t(ws->X, m, ws->n, ws->ldx, axi.data(), row.data(), 1);   // :66 X' axi
  ws->yax_rows.push_back(std::move(row));
  for (auto& r : ws->yay) r.resize(d + 1, 0.0);                  // :68 conservativeResize
  ws->yay.emplace_back(d + 1, 0.0);
  for (int64_t k = 0; k < d; ++k) {                              // :69-74
    const double v = dot8(xi, ws->a_basis[k].data(), m);
    ws->yay[d][k] = v;
    ws->yay[k][d] = v;
  }
  ws->yay[d][d] = dot8(axi.data(), xi, m);                       // :75
  ws->a_basis.push_back(std::move(axi));                         // :76-77
  ws->d = d + 1;                                                 // :81
  return ORC_OK;
}
int64_t orc_ws_d(orc_ws_t ws) { return ws->d; }
void orc_ws_col_sq(orc_ws_t ws, double* out) { std::copy(ws->col_sq.begin(), ws->col_sq.end(), out); }
void orc_ws_residual(orc_ws_t ws, double* out) {
  std::copy(ws->residual_sq.begin(), ws->residual_sq.end(), out);
}
void orc_ws_yax_row(orc_ws_t ws, int64_t k, double* out) {
  std::copy(ws->yax_rows[k].begin(), ws->yax_rows[k].end(), out);
}

int orc_ws_error_sq(orc_ws_t ws, int64_t j, const double* c, int64_t clen, double* out) {
  // workspace.cpp:84-99, identity quad = ||c||^2
  if (j < 0 || j >= ws->n) return fail(ORC_INDEX_OUT_OF_RANGE, "error_sq: column index out of range");
  if (clen != ws->d) return fail(ORC_DIMENSION_MISMATCH, "error_sq: coefficient length != d");
  double cross = 0.0;
  for (int64_t k = 0; k < ws->d; ++k) cross += c[k] * ws->yax_rows[k][j];
  double quad = 0.0;
  if (ws->diag.empty()) {
    for (int64_t k = 0; k < ws->d; ++k) quad += c[k] * c[k];  // :91 Y'AY = I
  } else {
    for (int64_t k = 0; k < ws->d; ++k) {                     // :93 c.dot(yay * c)
      double yc = 0.0;
      for (int64_t l = 0; l < ws->d; ++l) yc += ws->yay[k][l] * c[l];
      quad += c[k] * yc;
    }
  }
  const double e2 = ws->col_sq[j] - 2.0 * cross + quad;
  *out = e2 > 0.0 ? e2 : 0.0;
  return ORC_OK;
}

// residual_scan, general weight (workspace.cpp:114-122): error_sq of every
// column with c = T[:, j] (T row-major d x n).
int orc_ws_scan_T(orc_ws_t ws, const double* T, double* e_cur, int64_t* argmax) {
  double best = -1.0;
  int64_t arg = 0;
  std::vector<double> c(ws->d);
  for (int64_t j = 0; j < ws->n; ++j) {
    for (int64_t k = 0; k < ws->d; ++k) c[k] = T[k * ws->n + j];
    double e2;
    orc_ws_error_sq(ws, j, c.data(), ws->d, &e2);
    if (e2 > best) {
      best = e2;
      arg = j;
    }
  }
  *e_cur = std::sqrt(best > 0.0 ? best : 0.0);  // :123
  *argmax = arg;
  return ORC_OK;
}

int orc_ws_yay(orc_ws_t ws, double* out) {  // row-major d x d (zero-sized for identity)
  for (int64_t k = 0; k < (int64_t)ws->yay.size(); ++k)
    std::copy(ws->yay[k].begin(), ws->yay[k].end(), out + k * ws->d);
  return ORC_OK;
}

// rbd::decompose with a diagonal weight (decompose.cpp:53-111 with
// WeightSpec::diagonal, weight.cpp:11-21): Y and T stay Euclidean (mgs_project
// and T = xi'X are weight-free); the weight enters workspace_init/extend and
// the error_sq scan.
int orc_decompose_diag(const double* X, int64_t m, int64_t n, int64_t ldx, const double* diag,
                       int64_t diag_len, int64_t d_max, double eps_R, int start_kind,
                       int64_t start_column, uint64_t start_seed, int reorthogonalize,
                       double cfg_breakdown_tol, int64_t max_steps, double* Y, double* T,
                       int64_t* selected, double* history, int64_t* d_out) {
  // WeightSpec::diagonal (weight.cpp:11-17), constructed before decompose runs
  if (diag_len == 0) return fail(ORC_INVALID_ARGUMENT, "diagonal weight must be non-empty");
  for (int64_t i = 0; i < diag_len; ++i)
    if (!(diag[i] > 0.0) || !std::isfinite(diag[i]))
      return fail(ORC_INVALID_ARGUMENT, "diagonal weight entries must be strictly positive and finite");
  // validation, decompose.cpp:56-64 (same order)
  if (m < 1 || n < 1) return fail(ORC_INVALID_ARGUMENT, "decompose: matrix must be non-empty");
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i)
      if (!std::isfinite(X[i + j * ldx]))
        return fail(ORC_INVALID_ARGUMENT, "decompose: matrix has non-finite entries");
  if (d_max < 1 || d_max > n)
    return fail(ORC_INVALID_ARGUMENT, "decompose: d_max must satisfy 1 <= d_max <= n");
  if (!(eps_R >= 0.0)) return fail(ORC_INVALID_ARGUMENT, "decompose: eps_R must be >= 0");
  if (diag_len != m) return fail(ORC_INCOMPATIBLE_WEIGHT, "decompose: weight dimension != m");
  bool all_zero = true;
  for (int64_t j = 0; j < n && all_zero; ++j)
    for (int64_t i = 0; i < m; ++i)
      if (X[i + j * ldx] != 0.0) {
        all_zero = false;
        break;
      }
  if (all_zero) return fail(ORC_DEGENERATE_INPUT, "decompose: zero matrix, no basis can be built");
  double max_col_norm = 0.0;  // :70-74 (Euclidean column norms)
  for (int64_t j = 0; j < n; ++j)
    max_col_norm = std::max(max_col_norm, std::sqrt(sqnorm(X + j * ldx, m)));
  const double noise_floor =
      max_col_norm * std::sqrt(static_cast<double>(m)) * std::numeric_limits<double>::epsilon() * 16.0;
  const double breakdown_tol =
      std::max(cfg_breakdown_tol < 0.0 ? eps_R : cfg_breakdown_tol, noise_floor);
  orc_ws_t ws = orc_ws_init_diag(X, m, n, ldx, diag, diag_len);  // :81
  int64_t i;
  if (start_kind == 0) {
    if (start_column < 0 || start_column >= n) {
      orc_ws_free(ws);
      return fail(ORC_INDEX_OUT_OF_RANGE, "start column index out of range");
    }
    i = start_column;
  } else {
    i = orc_seeded_start(start_seed, n);
  }
  int64_t d = 0;
  double e_cur = std::numeric_limits<double>::infinity();
  std::vector<double> xi(m), row(n);
  while (d < d_max && e_cur > eps_R && d < max_steps) {  // :87
    double nrm;
    if (!orc_mgs_project(X + i * ldx, m, Y, d, m, breakdown_tol, reorthogonalize, xi.data(), &nrm))
      break;                                              // :90
    std::memcpy(Y + d * m, xi.data(), sizeof(double) * m);  // :92
    gemv_t(X, m, n, ldx, xi.data(), row.data(), 1);       // :93
    std::memcpy(T + d * n, row.data(), sizeof(double) * n);
    selected[d] = i;                                      // :94
    orc_ws_extend(ws, xi.data());                         // :95
    ++d;                                                  // :96
    int64_t arg;
    orc_ws_scan_T(ws, T, &e_cur, &arg);                   // :98 (T.topRows(d))
    history[d - 1] = e_cur;                               // :99
    i = arg;                                              // :101
  }
  orc_ws_free(ws);
  if (d == 0)
    return fail(ORC_DEGENERATE_INPUT, "decompose: start column is numerically zero, no basis built");
  *d_out = d;
  return ORC_OK;
}

int orc_ws_scan(orc_ws_t ws, double* e_cur, int64_t* argmax) {  // workspace.cpp:101-125
  double best = -1.0;
  int64_t arg = 0;
  for (int64_t j = 0; j < ws->n; ++j)
    if (ws->residual_sq[j] > best) {
      best = ws->residual_sq[j];
      arg = j;
    }
  *e_cur = std::sqrt(best > 0.0 ? best : 0.0);
  *argmax = arg;
  return ORC_OK;
}

// ---- project / reconstruct, decompose.cpp:113-123 ----
void orc_project(const double* Y, int64_t m, int64_t d, const double* v, double* c) {
  for (int64_t k = 0; k < d; ++k) c[k] = dot8(Y + k * m, v, m);
}
void orc_reconstruct(const double* Y, int64_t m, int64_t d, const double* c, double* v) {
  for (int64_t i = 0; i < m; ++i) v[i] = 0.0;
  for (int64_t k = 0; k < d; ++k) axpy(c[k], Y + k * m, v, m);
}
// Batched out-of-sample projection: Tn (d x N, column-major ld d) = Y' Xn and
// err_j = max(||x_j||^2 - ||t_j||^2, 0) (identity Eq.(3), workspace.cpp:88-97).
// Every Tn[k, j] is dot8(Y[:, k], x_j, m) — the per-vector project of
// decompose.cpp:113-117 — with the same 8 lane sums accumulated in the same row
// order; the loops are only tiled (row chunks x basis blocks x column blocks,
// lane sums carried across chunks) so that a config-4 batch (65536 x 16384
// against d = 512) finishes in seconds instead of re-reading Y per column.
void orc_project_batch(const double* Y, int64_t m, int64_t d, const double* Xn, int64_t N,
                       int64_t ldx, int nthreads, double* Tn, double* err) {
  constexpr int64_t JB = 32;    // columns per task
  constexpr int64_t KB = 128;    // basis vectors per task
  constexpr int64_t RC = 2048;  // rows per chunk (multiple of 8)
  const int64_t m8 = m - (m % 8);
  const int64_t nj = (N + JB - 1) / JB, nk = (d + KB - 1) / KB;
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1) if (nthreads > 1)
#endif
  for (int64_t task = 0; task < nj * nk; ++task) {
    const int64_t j0 = (task / nk) * JB, k0 = (task % nk) * KB;
    const int64_t jn = std::min(JB, N - j0), kn = std::min(KB, d - k0);
    std::vector<double> acc(static_cast<size_t>(KB * JB * 8), 0.0);
    for (int64_t r0 = 0; r0 < m8; r0 += RC) {
      const int64_t r1 = std::min(m8, r0 + RC);
      for (int64_t jj = 0; jj < jn; ++jj) {
        const double* x = Xn + (j0 + jj) * ldx;
        for (int64_t kk = 0; kk < kn; ++kk) {
          const double* y = Y + (k0 + kk) * m;
          double* s = acc.data() + (kk * JB + jj) * 8;
          double t[8];
          for (int l = 0; l < 8; ++l) t[l] = s[l];
          for (int64_t i = r0; i < r1; i += 8)
            for (int l = 0; l < 8; ++l) t[l] += y[i + l] * x[i + l];
          for (int l = 0; l < 8; ++l) s[l] = t[l];
        }
      }
    }
    for (int64_t jj = 0; jj < jn; ++jj) {
      const double* x = Xn + (j0 + jj) * ldx;
      for (int64_t kk = 0; kk < kn; ++kk) {
        const double* y = Y + (k0 + kk) * m;
        const double* s = acc.data() + (kk * JB + jj) * 8;
        double tail = 0.0;
        for (int64_t i = m8; i < m; ++i) tail += y[i] * x[i];
        Tn[(k0 + kk) + (j0 + jj) * d] =
            (((s[0] + s[4]) + (s[1] + s[5])) + ((s[2] + s[6]) + (s[3] + s[7]))) + tail;
      }
    }
  }
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads) schedule(static) if (nthreads > 1)
#endif
  for (int64_t j = 0; j < N; ++j) {
    if (!err) continue;
    double tt = 0.0;
    for (int64_t k = 0; k < d; ++k) {
      const double t = Tn[k + j * d];
      tt += t * t;
    }
    const double e = sqnorm(Xn + j * ldx, m) - tt;
    err[j] = e > 0.0 ? e : 0.0;
  }
  (void)nthreads;
}

// ---- Classifier::predict, batched (classify.cpp:22-34) ----
// c = Y'v (decompose.cpp:113-117), then the training column with the smallest
// (T[:,j] - c).squaredNorm(), strict '<' so the earliest column wins ties.
void orc_predict_batch(const double* Y, int64_t m, int64_t d, const double* T, int64_t n_tr,
                       const double* Qm, int64_t nq, int nthreads, int64_t* best_out,
                       double* dist_out) {
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads) schedule(static) if (nthreads > 1)
#endif
  for (int64_t q = 0; q < nq; ++q) {
    std::vector<double> c(d);
    for (int64_t k = 0; k < d; ++k) c[k] = dot8(Y + k * m, Qm + q * m, m);   // :23
    auto dist = [&](int64_t j) {                                                // :25,27
      double s = 0.0;
      for (int64_t k = 0; k < d; ++k) {
        const double df = T[k * n_tr + j] - c[k];
        s += df * df;
      }
      return s;
    };
    int64_t best = 0;
    double best_dist = dist(0);
    for (int64_t j = 1; j < n_tr; ++j) {                                        // :26-32
      const double dj = dist(j);
      if (dj < best_dist) {
        best_dist = dj;
        best = j;
      }
    }
    best_out[q] = best;
    if (dist_out) dist_out[q] = best_dist;
  }
  (void)nthreads;
}

// gen_labeled_blobs (datasets.cpp:67-97): unit-norm Gaussian class centres plus
// spread * N(0,1) per sample, classes in order; samples dim x (n_classes*per_class).
int orc_gen_labeled_blobs(int n_classes, int per_class, int dim, double spread, uint64_t seed,
                          double* samples, int* labels) {
  if (n_classes < 1 || per_class < 1 || dim < 1) return fail(ORC_INVALID_ARGUMENT, "blob counts must be >= 1");
  if (!(spread >= 0.0)) return fail(ORC_INVALID_ARGUMENT, "spread must be >= 0");
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  std::vector<double> centers(static_cast<size_t>(dim) * n_classes);
  for (int c = 0; c < n_classes; ++c) {
    std::vector<double> g(dim);
    for (int i = 0; i < dim; ++i) g[i] = gauss(rng);
    double nrm = 0.0;   // Eigen norm(): sqrt of the squared norm
    for (int i = 0; i < dim; ++i) nrm += g[i] * g[i];
    nrm = std::sqrt(nrm);
    for (int i = 0; i < dim; ++i)
      centers[i + static_cast<size_t>(c) * dim] = nrm > 0.0 ? g[i] / nrm : (i == 0 ? 1.0 : 0.0);
  }
  int64_t col = 0;
  for (int c = 0; c < n_classes; ++c)
    for (int k = 0; k < per_class; ++k, ++col) {
      for (int i = 0; i < dim; ++i)
        samples[i + col * dim] = centers[i + static_cast<size_t>(c) * dim] + spread * gauss(rng);
      labels[col] = c;
    }
  return ORC_OK;
}

// ---- fixtures ----
void orc_random_matrix(int64_t m, int64_t n, uint64_t seed, double* out) {
  // helpers.hpp:14-21 / acceptance.cpp:56-63: column-major fill
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) out[i + j * m] = gauss(rng);
}

void orc_random_positive(int64_t n, uint64_t seed, double* out) {
  // helpers.hpp:28-34: U[0.5, 3.0) draws
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.5, 3.0);
  for (int64_t i = 0; i < n; ++i) out[i] = u(rng);
}

void orc_random_low_rank(int64_t m, int64_t n, int64_t r, uint64_t seed, double* out) {
  // helpers.hpp:23-26: random_matrix(m,r,seed) * random_matrix(r,n,seed+1)
  std::vector<double> a(m * r), b(r * n);
  orc_random_matrix(m, r, seed, a.data());
  orc_random_matrix(r, n, seed + 1, b.data());
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      double s = 0.0;
      for (int64_t k = 0; k < r; ++k) s += a[i + k * m] * b[k + j * r];
      out[i + j * m] = s;
    }
}

static double eval_function(int f, double x, double y) {  // datasets.cpp:15-45
  const double pi = 3.14159265358979323846;
  switch (f) {
    case 0:
      return std::sin(pi * x) * std::cos(pi * y);
    case 1:
      return eval_function(0, x, y) + 0.1 * std::sin(10.0 * pi * x) * std::cos(10.0 * pi * y);
    case 2:
      return eval_function(1, x, y) + 0.01 * std::sin(100.0 * pi * x) * std::cos(100.0 * pi * y);
    case 3: {
      const double f1 = std::sin(pi * (x + 2.0 * y)) * std::cos(pi * (2.0 * x - y));
      const double f2 = std::sin(10.0 * pi * (x - 3.0 * y)) * std::cos(10.0 * pi * (3.0 * x + y));
      const double f3 = std::sin(3.0 * pi * x * x * y) *
                        std::cos(6.0 * pi * std::sqrt(std::abs(x)) / (y + 2.0));
      return 0.6 * f1 + 0.1 * f2 + 0.01 * f3;
    }
  }
  return 0.0;
}

int orc_gen_grid_matrix(int fid, int64_t n_points, double* out) {  // datasets.cpp:47-65
  if (n_points < 2) return fail(ORC_INVALID_ARGUMENT, "grid needs at least 2 points per axis");
  const int64_t n = n_points;
  const double hx = 2.0 / static_cast<double>(n - 1);
  const double hy = 2.0 / static_cast<double>(n - 1);
  for (int64_t j = 0; j < n; ++j) {
    const double y = -1.0 + static_cast<double>(j) * hy;
    for (int64_t i = 0; i < n; ++i) {
      const double x = -1.0 + static_cast<double>(i) * hx;
      out[i + j * n] = eval_function(fid, x, y);
    }
  }
  return ORC_OK;
}

int64_t orc_acceptance3_count(void) {
  // acceptance.cpp:185-231: restates the harness's RNG consumption. Every
  // instance is a seeded Gaussian matrix (full rank), so model.d equals the
  // drawn d; the count is sum of n over the 200 instances.
  std::mt19937_64 rng(314159);
  int64_t checked = 0;
  for (int instance = 0; instance < 200; ++instance) {
    const int64_t m = 5 + static_cast<int64_t>(rng() % 36);
    const int64_t n = 4 + static_cast<int64_t>(rng() % 27);
    const int64_t d_cap = std::min<int64_t>({10, m, n});
    const int64_t d = 1 + static_cast<int64_t>(rng() % d_cap);
    const int kind = instance % 3;
    if (kind == 1) {
      std::uniform_real_distribution<double> u(0.25, 4.0);
      for (int64_t i = 0; i < m; ++i) (void)u(rng);
    } else if (kind == 2) {
      (void)rng();  // random_spd(m, rng())
    }
    std::vector<double> x(m * n);
    orc_random_matrix(m, n, rng(), x.data());
    std::vector<double> Y(m * d), T(d * n), hist(d);
    std::vector<int64_t> sel(d);
    int64_t got = 0;
    orc_decompose(x.data(), m, n, m, d, 0.0, 0, 0, 0, 0, -1.0, 1, Y.data(), T.data(), sel.data(),
                  hist.data(), &got);
    std::uniform_real_distribution<double> shift(-0.5, 0.5);
    for (int64_t j = 0; j < n; ++j) {
      if (instance % 2 == 1)
        for (int64_t k = 0; k < got; ++k) (void)shift(rng);
      ++checked;
    }
  }
  return checked;
}

}  // extern "C"
