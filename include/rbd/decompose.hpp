// rbd/decompose.hpp — drop-in for proj/include/rbd/decompose.hpp:13-79 on B200:
// same names, fields, defaults and error types; the work runs on the GPU
// through the C ABI (include/rbd_cuda.h). Link with librbd_b200.so.
#ifndef RBD_B200_DECOMPOSE_HPP
#define RBD_B200_DECOMPOSE_HPP

#include <cstdint>
#include <mutex>
#include <optional>
#include <vector>

#include "rbd/errors.hpp"
#include "rbd/types.hpp"
#include "rbd/weight.hpp"
#include "rbd_cuda.h"

namespace rbd {

struct StartSpec {                                   // decompose.hpp:14-23
  enum class Kind { fixed_column, seeded_random };
  static StartSpec column(Index i) { return {Kind::fixed_column, i, 0}; }
  static StartSpec seeded(std::uint64_t s) { return {Kind::seeded_random, 0, s}; }
  Kind kind = Kind::fixed_column;
  Index column_index = 0;
  std::uint64_t seed = 0;
};

struct RbdConfig {                                   // decompose.hpp:25-36
  Index d_max = 1;
  double eps_R = 0.0;
  StartSpec start{};
  WeightSpec weight{};
  bool reorthogonalize = false;
  double breakdown_tol = -1.0;
};

namespace detail {
inline rbd_ctx_t context();
inline void check(int status);

// A model's device-resident Y (rbd_model_t), created by the first project /
// reconstruct and reused by the later ones, so the reference's per-vector
// callers (classify.cpp:22-23, tools/main.cpp:149-158) upload Y once instead
// of per call. Copies of a model start with an empty cache; the key (Y's
// buffer and shape) rebuilds it if Y was replaced.
class ResidentCache {
 public:
  ResidentCache() = default;
  ResidentCache(const ResidentCache&) {}
  ResidentCache& operator=(const ResidentCache&) {
    std::lock_guard<std::mutex> g(mu_);
    drop();
    return *this;
  }
  ~ResidentCache() { drop(); }
  rbd_model_t get(const Matrix& Y, Index d) const {
    std::lock_guard<std::mutex> g(mu_);
    if (h_ && key_ == Y.data() && m_ == Y.rows() && d_ == d) return h_;
    drop();
    rbd_model_t h = nullptr;
    check(rbd_model_create(context(), Y.rows(), d, d, Y.data(), Y.rows(), nullptr, 0, nullptr,
                           0.0, &h));
    h_ = h;
    key_ = Y.data();
    m_ = Y.rows();
    d_ = d;
    return h_;
  }

 private:
  void drop() const {
    if (h_) rbd_model_free(h_);
    h_ = nullptr;
  }
  mutable std::mutex mu_;
  mutable rbd_model_t h_ = nullptr;
  mutable const double* key_ = nullptr;
  mutable Index m_ = 0, d_ = 0;
};
}  // namespace detail

struct RbdModel {                                    // decompose.hpp:39-46
  Matrix Y;                                          // m x d
  Matrix T;                                          // d x n
  std::vector<Index> selected;
  std::vector<double> residual_history;
  Index d = 0;
  WeightSpec weight{};
  detail::ResidentCache resident{};                  // B200: device copy of Y (not in the reference)
};

struct MgsResult {                                   // decompose.hpp:48-51
  Vector xi;
  double residual_norm;
};

namespace detail {
// One context per host thread (rbd_cuda.h threading contract).
inline rbd_ctx_t context() {
  struct Holder {
    rbd_ctx_t c = nullptr;
    ~Holder() {
      if (c) rbd_ctx_destroy(c);
    }
  };
  thread_local Holder h;
  if (!h.c) check(rbd_ctx_create(0, &h.c));
  return h.c;
}
}  // namespace detail

inline std::optional<MgsResult> mgs_project(const VectorRef& v, const MatrixRef& basis,
                                            double breakdown_tol, bool reorthogonalize = false) {
  if (basis.cols() > 0 && basis.rows() != v.size())
    throw DimensionMismatch("mgs_project: vector length != basis row count");
  Vector xi(v.size());
  double norm = 0.0;
  int ok = 0;
  detail::check(rbd_mgs_project_host(detail::context(), v.data(), v.size(), basis.data(),
                                     basis.cols(), basis.rows(), breakdown_tol,
                                     reorthogonalize ? 1 : 0, xi.data(), &norm, &ok));
  if (!ok) return std::nullopt;
  return MgsResult{std::move(xi), norm};
}

namespace detail {
inline rbd_config_t to_c(const RbdConfig& cfg) {
  rbd_config_t c;
  rbd_config_default(&c);
  c.d_max = cfg.d_max;
  c.eps_R = cfg.eps_R;
  c.start_kind = cfg.start.kind == StartSpec::Kind::seeded_random ? RBD_START_SEEDED_RANDOM
                                                                  : RBD_START_FIXED_COLUMN;
  c.start_column = cfg.start.column_index;
  c.start_seed = cfg.start.seed;
  c.reorthogonalize = cfg.reorthogonalize ? 1 : 0;
  c.breakdown_tol = cfg.breakdown_tol;
  c.weight_kind = static_cast<int32_t>(cfg.weight.kind());
  c.weight_dim = cfg.weight.dim();
  return c;
}

// RbdModel from the C ABI's outputs (Y column-major m x cap, T row-major cap x n).
inline RbdModel to_model(const rbd_result_t& r, Index m, Index n, const std::vector<double>& Yb,
                         const std::vector<double>& Tb, const std::vector<int64_t>& sel,
                         const std::vector<double>& hist, const WeightSpec& weight) {
  RbdModel model;
  model.d = r.d;
  model.weight = weight;
  model.Y = Matrix(m, r.d);
  for (Index j = 0; j < r.d; ++j)
    for (Index i = 0; i < m; ++i) model.Y(i, j) = Yb[static_cast<size_t>(i + j * m)];
  model.T = Matrix(r.d, n);
  for (Index k = 0; k < r.d; ++k)
    for (Index j = 0; j < n; ++j) model.T(k, j) = Tb[static_cast<size_t>(k * n + j)];
  model.selected.assign(sel.begin(), sel.begin() + r.d);
  model.residual_history.assign(hist.begin(), hist.begin() + r.d);
  return model;
}
}  // namespace detail

// A caller's loop of decompose() over matrices of one shape and config, with
// the upload of matrix i+1 overlapping matrix i's greedy loop
// (rbd_decompose_host_many; identity weight). Same results as decompose() on
// each matrix.
inline std::vector<RbdModel> decompose_many(const std::vector<Matrix>& xs, const RbdConfig& cfg) {
  std::vector<RbdModel> out;
  if (xs.empty()) return out;
  if (cfg.weight.kind() != WeightKind::identity)
    throw InvalidArgument("decompose_many: identity weight only");
  const Index m = xs[0].rows(), n = xs[0].cols();
  for (const Matrix& x : xs)
    if (x.rows() != m || x.cols() != n) throw InvalidArgument("decompose_many: matrices must be of one shape");
  const rbd_config_t c = detail::to_c(cfg);
  const Index cap = std::max<Index>(1, std::min<Index>(cfg.d_max, std::max<Index>(n, 1)));
  const size_t cnt = xs.size();
  std::vector<std::vector<double>> Yb(cnt), Tb(cnt), hist(cnt);
  std::vector<std::vector<int64_t>> sel(cnt);
  std::vector<const double*> xp(cnt);
  std::vector<double*> yp(cnt), tp(cnt), hp(cnt);
  std::vector<int64_t*> sp(cnt);
  std::vector<rbd_result_t> r(cnt);
  for (size_t i = 0; i < cnt; ++i) {
    Yb[i].resize(static_cast<size_t>(std::max<Index>(m, 1) * cap));
    Tb[i].resize(static_cast<size_t>(cap * std::max<Index>(n, 1)));
    sel[i].resize(static_cast<size_t>(cap));
    hist[i].resize(static_cast<size_t>(cap));
    xp[i] = xs[i].data();
    yp[i] = Yb[i].data();
    tp[i] = Tb[i].data();
    sp[i] = sel[i].data();
    hp[i] = hist[i].data();
  }
  detail::check(rbd_decompose_host_many(detail::context(), static_cast<int64_t>(cnt), xp.data(), m, n,
                                        std::max<Index>(m, 1), &c, yp.data(), tp.data(), sp.data(),
                                        hp.data(), r.data()));
  out.reserve(cnt);
  for (size_t i = 0; i < cnt; ++i)
    out.push_back(detail::to_model(r[i], m, n, Yb[i], Tb[i], sel[i], hist[i], cfg.weight));
  return out;
}

inline RbdModel decompose(const Matrix& x, const RbdConfig& cfg) {
  const rbd_config_t c = detail::to_c(cfg);
  const Index m = x.rows(), n = x.cols();
  const Index cap = std::max<Index>(1, std::min<Index>(cfg.d_max, std::max<Index>(n, 1)));
  std::vector<double> Yb(static_cast<size_t>(std::max<Index>(m, 1) * cap));
  std::vector<double> Tb(static_cast<size_t>(cap * std::max<Index>(n, 1)));
  std::vector<int64_t> sel(static_cast<size_t>(cap));
  std::vector<double> hist(static_cast<size_t>(cap));
  rbd_result_t r{};
  if (cfg.weight.kind() == WeightKind::diagonal) {
    const Vector& dg = cfg.weight.diagonal_values();
    detail::check(rbd_decompose_diag_host(detail::context(), x.data(), m, n,
                                          std::max<Index>(m, 1), &c, dg.data(), dg.size(),
                                          Yb.data(), Tb.data(), sel.data(), hist.data(), &r));
  } else {
    detail::check(rbd_decompose_host(detail::context(), x.data(), m, n, std::max<Index>(m, 1),
                                     &c, Yb.data(), Tb.data(), sel.data(), hist.data(), &r));
  }
  return detail::to_model(r, m, n, Yb, Tb, sel, hist, cfg.weight);   // device T is row-major
}

inline Vector project(const RbdModel& model, const VectorRef& v) {     // decompose.cpp:113-117
  if (v.size() != model.Y.rows()) throw DimensionMismatch("project: vector length != m");
  Vector c(model.d);
  if (model.d == 0) return c;
  detail::check(rbd_project_model(detail::context(), model.resident.get(model.Y, model.d),
                                  v.data(), 1, v.size(), c.data(), nullptr));
  return c;
}

inline Vector reconstruct(const RbdModel& model, const VectorRef& c) { // decompose.cpp:119-123
  if (c.size() != model.d) throw DimensionMismatch("reconstruct: coefficient length != d");
  Vector v(model.Y.rows());
  if (model.d == 0) return v;
  detail::check(rbd_reconstruct_model(detail::context(), model.resident.get(model.Y, model.d),
                                      c.data(), 1, v.data()));
  return v;
}

inline Matrix compress_matrix(const RbdModel& model) {                 // decompose.cpp:125
  Matrix out(model.Y.rows(), model.T.cols());
  if (model.d == 0 || model.T.cols() == 0) return out;
  detail::check(rbd_compress_host(detail::context(), model.Y.data(), model.Y.rows(), model.d,
                                  model.T.data(), model.T.cols(), out.data()));
  return out;
}

}  // namespace rbd

#endif
