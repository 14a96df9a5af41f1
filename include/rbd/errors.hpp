// rbd/errors.hpp — the reference's exception hierarchy
// (proj/include/rbd/errors.hpp:9-77), plus the mapping from
// the C ABI status codes (include/rbd_cuda.h).
#ifndef RBD_B200_ERRORS_HPP
#define RBD_B200_ERRORS_HPP

#include <cstdlib>
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
class UnsupportedFormat : public Error { public: using Error::Error; };
class IoError : public Error { public: using Error::Error; };
class ParseError : public Error {                   // errors.hpp:64-77
 public:
  ParseError(const std::string& path, long line, const std::string& what)
      : Error(path + ":" + std::to_string(line) + ": " + what), path_(path), line_(line) {}
  explicit ParseError(const std::string& full) : Error(full), line_(0) {
    // "path:line: what" as produced by the library
    const auto a = full.find(':');
    if (a != std::string::npos) {
      path_ = full.substr(0, a);
      line_ = std::strtol(full.c_str() + a + 1, nullptr, 10);
    }
  }
  const std::string& path() const { return path_; }
  long line() const { return line_; }

 private:
  std::string path_;
  long line_;
};

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
    case RBD_ERR_UNSUPPORTED_FORMAT: throw UnsupportedFormat(msg);
    case RBD_ERR_IO: throw IoError(msg);
    case RBD_ERR_PARSE: throw ParseError(msg);
    default: throw Error(msg);
  }
}
}  // namespace detail

}  // namespace rbd

#endif
