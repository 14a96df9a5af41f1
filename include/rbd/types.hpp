// rbd/types.hpp — the reference's Eigen aliases (proj/include/rbd/types.hpp:10-16)
// re-expressed without Eigen: an owning column-major dense matrix and vector
// with the member functions the hot-path callers use.
#ifndef RBD_B200_TYPES_HPP
#define RBD_B200_TYPES_HPP

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <initializer_list>
#include <stdexcept>
#include <vector>

namespace rbd {

using Index = std::ptrdiff_t;   // Eigen::Index

class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n) : v_(static_cast<size_t>(n), 0.0) {}
  Vector(std::initializer_list<double> il) : v_(il) {}
  static Vector Zero(Index n) { return Vector(n); }
  static Vector Ones(Index n) {
    Vector v(n);
    for (auto& x : v.v_) x = 1.0;
    return v;
  }
  Index size() const { return static_cast<Index>(v_.size()); }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator[](Index i) { return v_[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return v_[static_cast<size_t>(i)]; }
  double& operator()(Index i) { return v_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<size_t>(i)]; }
  double squaredNorm() const {
    double s = 0.0;
    for (double x : v_) s += x * x;
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  double dot(const Vector& o) const {
    double s = 0.0;
    for (size_t i = 0; i < v_.size(); ++i) s += v_[i] * o.v_[i];
    return s;
  }

 private:
  std::vector<double> v_;
};

// Column-major m x n, leading dimension m (Eigen::MatrixXd layout).
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index m, Index n) : m_(m), n_(n), a_(static_cast<size_t>(m * n), 0.0) {}
  static Matrix Zero(Index m, Index n) { return Matrix(m, n); }
  static Matrix Identity(Index m, Index n) {
    Matrix I(m, n);
    for (Index i = 0; i < std::min(m, n); ++i) I(i, i) = 1.0;
    return I;
  }
  Index rows() const { return m_; }
  Index cols() const { return n_; }
  Index size() const { return m_ * n_; }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }
  double& operator()(Index i, Index j) { return a_[static_cast<size_t>(i + j * m_)]; }
  double operator()(Index i, Index j) const { return a_[static_cast<size_t>(i + j * m_)]; }
  Vector col(Index j) const {
    Vector v(m_);
    for (Index i = 0; i < m_; ++i) v[i] = (*this)(i, j);
    return v;
  }
  void set_col(Index j, const Vector& v) {
    for (Index i = 0; i < m_; ++i) (*this)(i, j) = v[i];
  }
  Matrix leftCols(Index k) const {
    Matrix r(m_, k);
    for (Index j = 0; j < k; ++j)
      for (Index i = 0; i < m_; ++i) r(i, j) = (*this)(i, j);
    return r;
  }
  bool operator==(const Matrix& o) const { return m_ == o.m_ && n_ == o.n_ && a_ == o.a_; }

 private:
  Index m_ = 0, n_ = 0;
  std::vector<double> a_;
};

using MatrixRef = const Matrix&;
using VectorRef = const Vector&;

}  // namespace rbd

#endif
