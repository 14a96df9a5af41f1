// rbd/workspace.hpp — ErrorWorkspace API (proj/include/rbd/workspace.hpp:18-54),
// identity and diagonal weights, on the B200 (the workspace owns a device copy
// of X).
#ifndef RBD_B200_WORKSPACE_HPP
#define RBD_B200_WORKSPACE_HPP

#include <memory>
#include <vector>

#include "rbd/decompose.hpp"

namespace rbd {

struct ErrorWorkspace {
  WeightKind kind = WeightKind::identity;
  Index m = 0, n = 0, d = 0;
  std::shared_ptr<rbd_ws_s> h;
  Vector col_sq() const {
    Vector v(n);
    detail::check(rbd_ws_read(h.get(), v.data(), nullptr, nullptr));
    return v;
  }
  Vector residual_sq() const {
    Vector v(n);
    detail::check(rbd_ws_read(h.get(), nullptr, v.data(), nullptr));
    return v;
  }
};

struct ScanResult {
  double e_cur = 0.0;
  Index argmax = 0;
};

inline ErrorWorkspace workspace_init(const Matrix& x, const WeightSpec& a) {   // workspace.cpp:9-41
  if (!a.compatible_with(x.rows()))
    throw IncompatibleWeight("weight dimension does not match matrix rows");
  if (a.kind() == WeightKind::sparse_spd)
    throw InvalidArgument("workspace_init: sparse SPD weights are out of scope on the B200 path");
  ErrorWorkspace ws;
  ws.kind = a.kind();
  ws.m = x.rows();
  ws.n = x.cols();
  rbd_ws_t h = nullptr;
  if (a.kind() == WeightKind::diagonal)
    detail::check(rbd_ws_init_diag_host(detail::context(), x.data(), ws.m, ws.n, ws.m, ws.n,
                                        a.diagonal_values().data(), a.diagonal_values().size(),
                                        &h));
  else
    detail::check(rbd_ws_init_host(detail::context(), x.data(), ws.m, ws.n, ws.m, ws.n, &h));
  ws.h = std::shared_ptr<rbd_ws_s>(h, [](rbd_ws_s* p) { rbd_ws_destroy(p); });
  return ws;
}

inline void workspace_extend(ErrorWorkspace& ws, const VectorRef& xi, const Matrix& x,
                             const WeightSpec&) {                            // workspace.cpp:43-60
  if (xi.size() != ws.m || x.rows() != ws.m || x.cols() != ws.n)
    throw DimensionMismatch("workspace_extend: dimensions changed since init");
  detail::check(rbd_ws_extend_host(ws.h.get(), xi.data()));
  ws.d = rbd_ws_d(ws.h.get());
}

inline double error_sq(const ErrorWorkspace& ws, Index j, const VectorRef& c) {  // :84-99
  double out = 0.0;
  detail::check(rbd_ws_error_sq(ws.h.get(), j, c.data(), c.size(), &out));
  return out;
}

inline ScanResult residual_scan(const ErrorWorkspace& ws, const MatrixRef& t) {  // :101-125
  if (t.rows() != ws.d || t.cols() != ws.n)
    throw DimensionMismatch("residual_scan: T shape does not match workspace");
  ScanResult r;
  int64_t arg = 0;
  if (ws.kind == WeightKind::identity) {
    detail::check(rbd_ws_scan(ws.h.get(), &r.e_cur, &arg));
  } else {   // general weight: error_sq of every column with c = T[:, j]
    std::vector<double> trow(static_cast<size_t>(ws.d * ws.n));
    for (Index k = 0; k < ws.d; ++k)
      for (Index j = 0; j < ws.n; ++j) trow[static_cast<size_t>(k * ws.n + j)] = t(k, j);
    detail::check(rbd_ws_scan_T_host(ws.h.get(), trow.data(), &r.e_cur, &arg));
  }
  r.argmax = arg;
  return r;
}

}  // namespace rbd

#endif
