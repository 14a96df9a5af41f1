// rbd/errors.hpp — the reference's exception hierarchy
// (proj/include/rbd/errors.hpp:9-77), hot-path subset, plus the mapping from
// the C ABI status codes (include/rbd_cuda.h).
#ifndef RBD_B200_ERRORS_HPP
#define RBD_B200_ERRORS_HPP

#include <stdexcept>
#include <string>

#include "rbd_cuda.h"

namespace rbd {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DimensionMismatch : public Error { public: using Error::Error; };
class IncompatibleWeight : public Error { public: using Error::Error; };
class DegenerateInput : public Error { public: using Error::Error; };
class NotPositive : public Error { public: using Error::Error; };
class IndexOutOfRange : public Error { public: using Error::Error; };
class NoConvergence : public Error { public: using Error::Error; };
class InvalidArgument : public Error { public: using Error::Error; };

namespace detail {
inline void check(int status) {
  if (status == RBD_OK) return;
  const std::string msg = rbd_last_error();
  switch (status) {
    case RBD_ERR_INVALID_ARGUMENT: throw InvalidArgument(msg);
    case RBD_ERR_INCOMPATIBLE_WEIGHT: throw IncompatibleWeight(msg);
    case RBD_ERR_DEGENERATE_INPUT: throw DegenerateInput(msg);
    case RBD_ERR_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(msg);
    case RBD_ERR_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case RBD_ERR_NOT_POSITIVE: throw NotPositive(msg);
    case RBD_ERR_NO_CONVERGENCE: throw NoConvergence(msg);
    default: throw Error(msg);
  }
}
}  // namespace detail

}  // namespace rbd

#endif
