// tsylv drop-in (B200 build) — column-major dense matrix (the BLAS/LAPACK
// layout of the reference's Matrix<T>, matrix.hpp:16-97) and the exact
// structural predicates the reduced-form solvers validate with
// (matrix.hpp:152-172; no tolerance: LAPACK writes exact zeros).
#pragma once
#include <cmath>
#include <cstddef>
#include <vector>

#include "tsylv/errors.hpp"
#include "tsylv/scalar.hpp"

namespace tsylv {

template <typename T>
class Matrix {
 public:
  Matrix() = default;
  Matrix(int r, int c) : r_(r), c_(c), v_(checked(r, c), T{}) {}
  Matrix(int r, int c, std::vector<T> v) : r_(r), c_(c), v_(std::move(v)) {
    if (v_.size() != checked(r, c)) throw dimension_error("Matrix: data size does not match shape");
  }
  static Matrix identity(int n) {
    Matrix m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = T(1);
    return m;
  }
  int rows() const noexcept { return r_; }
  int cols() const noexcept { return c_; }
  std::size_t size() const noexcept { return v_.size(); }
  bool empty() const noexcept { return v_.empty(); }
  T* data() noexcept { return v_.data(); }
  const T* data() const noexcept { return v_.data(); }
  T& operator()(int i, int j) { return v_[i + static_cast<std::size_t>(j) * r_]; }
  const T& operator()(int i, int j) const { return v_[i + static_cast<std::size_t>(j) * r_]; }

  Matrix block(int r0, int r1, int c0, int c1) const {
    if (r0 < 0 || c0 < 0 || r1 > r_ || c1 > c_ || r1 < r0 || c1 < c0)
      throw dimension_error("Matrix::block: range out of bounds");
    Matrix b(r1 - r0, c1 - c0);
    for (int j = c0; j < c1; ++j)
      for (int i = r0; i < r1; ++i) b(i - r0, j - c0) = (*this)(i, j);
    return b;
  }
  double frobenius_norm() const {
    double s = 0;
    for (const T& x : v_) s += abs_squared(x);
    return std::sqrt(s);
  }
  Matrix& operator*=(T s) {
    for (T& x : v_) x *= s;
    return *this;
  }

 private:
  static std::size_t checked(int r, int c) {
    if (r < 0 || c < 0) throw dimension_error("Matrix: negative dimension");
    return static_cast<std::size_t>(r) * c;
  }
  int r_ = 0, c_ = 0;
  std::vector<T> v_;
};

template <typename T>
Matrix<T> transposed(const Matrix<T>& a) {
  Matrix<T> t(a.cols(), a.rows());
  for (int j = 0; j < a.cols(); ++j)
    for (int i = 0; i < a.rows(); ++i) t(j, i) = a(i, j);
  return t;
}

// Elementwise conjugate and conjugate transpose (matrix.hpp:120-148; the
// identity / plain transpose for T = double).
template <typename T>
Matrix<T> conjugated(const Matrix<T>& a) {
  Matrix<T> c = a;
  for (std::size_t i = 0; i < c.size(); ++i) c.data()[i] = conjugate(c.data()[i]);
  return c;
}
template <typename T>
Matrix<T> adjoint(const Matrix<T>& a) {
  return conjugated(transposed(a));
}

template <typename T>
bool is_upper_triangular(const Matrix<T>& a) {
  for (int j = 0; j < a.cols(); ++j)
    for (int i = j + 1; i < a.rows(); ++i)
      if (a(i, j) != T{}) return false;
  return true;
}

// 1x1/2x2 diagonal blocks only: nothing below the first sub-diagonal and no
// two adjacent sub-diagonal entries.
template <typename T>
bool is_upper_quasi_triangular(const Matrix<T>& a) {
  const int n = a.rows();
  if (n != a.cols()) return false;
  for (int j = 0; j < n; ++j) {
    for (int i = j + 2; i < n; ++i)
      if (a(i, j) != T{}) return false;
    if (j + 2 < n && a(j + 1, j) != T{} && a(j + 2, j + 1) != T{}) return false;
  }
  return true;
}

}  // namespace tsylv
