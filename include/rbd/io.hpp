// rbd/io.hpp — the reference's model container API (proj/include/rbd/io.hpp:51-64)
// over the C ABI (rbd_model_write / rbd_model_read).
#ifndef RBD_B200_IO_HPP
#define RBD_B200_IO_HPP

#include <filesystem>
#include <vector>

#include "rbd/decompose.hpp"
#include "rbd/errors.hpp"
#include "rbd_cuda.h"

namespace rbd {

/// "RBD1" | u64 m, n, d | weight tag | f64 Y col-major | f64 T row-major |
/// f64 eps_R | f64 residual_history[d] | (tag 1) f64 diag[m]; little-endian.
inline void write_model(const RbdModel& model, double eps_r, const std::filesystem::path& path) {
  const Index m = model.Y.rows(), n = model.T.cols(), d = model.d;
  if (model.Y.cols() != d || model.T.rows() != d ||
      static_cast<Index>(model.residual_history.size()) != d)
    throw DimensionMismatch("write_model: inconsistent model shapes");
  std::vector<double> trow(static_cast<size_t>(d * n));   // the container stores T row-major
  for (Index k = 0; k < d; ++k)
    for (Index j = 0; j < n; ++j) trow[static_cast<size_t>(k * n + j)] = model.T(k, j);
  const int tag = static_cast<int>(model.weight.kind());
  detail::check(rbd_model_write(nullptr, path.c_str(), m, n, d, model.Y.data(), m, trow.data(),
                                eps_r, model.residual_history.data(), tag,
                                tag == 1 ? model.weight.diagonal_values().data() : nullptr));
}

struct LoadedModel {
  RbdModel model;
  double eps_r = 0.0;
};

inline LoadedModel read_model(const std::filesystem::path& path) {
  int64_t m = 0, n = 0, d = 0;
  int tag = 0;
  detail::check(rbd_model_read_header(path.c_str(), &m, &n, &d, &tag));
  LoadedModel out;
  out.model.d = d;
  out.model.Y = Matrix(m, d);
  std::vector<double> trow(static_cast<size_t>(d * n));
  out.model.residual_history.resize(static_cast<size_t>(d));
  Vector diag(tag == 1 ? m : 0);
  detail::check(rbd_model_read(nullptr, path.c_str(), out.model.Y.data(), m, trow.data(),
                               &out.eps_r, out.model.residual_history.data(),
                               tag == 1 ? diag.data() : nullptr));
  out.model.T = Matrix(d, n);
  for (Index k = 0; k < d; ++k)
    for (Index j = 0; j < n; ++j) out.model.T(k, j) = trow[static_cast<size_t>(k * n + j)];
  if (tag == 1) out.model.weight = WeightSpec::diagonal(std::move(diag));
  else if (tag == 2) out.model.weight = WeightSpec::sparse_external();
  return out;
}

}  // namespace rbd

#endif
