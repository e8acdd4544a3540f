// tsylv drop-in (B200 build) — dense order-d tensor, mode 0 fastest
// (offset i0 + i1*n0 + ..., reference tensor.hpp:19-27), and the mode product
// Y = X x_m A (Y_(m) = A X_(m), tensor.hpp:184-231), which here runs on the
// DMMA batched GEMM of the GPU library (tsg_mode_multiply).
#pragma once
#include <cmath>
#include <cstddef>
#include <string>
#include <vector>

#include "tsylv/errors.hpp"
#include "tsylv/gpu.hpp"
#include "tsylv/matrix.hpp"

namespace tsylv {

template <typename T>
class Tensor {
 public:
  Tensor() = default;
  explicit Tensor(std::vector<int> dims) : dims_(std::move(dims)), v_(count(dims_), T{}) {}
  Tensor(std::vector<int> dims, std::vector<T> v) : dims_(std::move(dims)), v_(std::move(v)) {
    if (v_.size() != count(dims_)) throw dimension_error("Tensor: data size does not match dims");
  }
  int order() const noexcept { return static_cast<int>(dims_.size()); }
  const std::vector<int>& dims() const noexcept { return dims_; }
  int dim(int m) const {
    if (m < 0 || m >= order()) throw dimension_error("Tensor: mode out of range");
    return dims_[m];
  }
  std::size_t size() const noexcept { return v_.size(); }
  T* data() noexcept { return v_.data(); }
  const T* data() const noexcept { return v_.data(); }
  const std::vector<T>& values() const noexcept { return v_; }
  std::vector<T> take_values() && { return std::move(v_); }
  double frobenius_norm() const {
    double s = 0;
    for (const T& x : v_) s += abs_squared(x);
    return std::sqrt(s);
  }
  template <typename... I>
  T& operator()(I... idx) {
    return v_[offset({static_cast<int>(idx)...})];
  }
  template <typename... I>
  const T& operator()(I... idx) const {
    return v_[offset({static_cast<int>(idx)...})];
  }
  std::size_t offset(const std::vector<int>& ix) const {
    if (static_cast<int>(ix.size()) != order()) throw dimension_error("Tensor: index order mismatch");
    std::size_t o = 0, s = 1;
    for (int m = 0; m < order(); ++m) {
      if (ix[m] < 0 || ix[m] >= dims_[m]) throw dimension_error("Tensor: index out of range");
      o += s * static_cast<std::size_t>(ix[m]);
      s *= static_cast<std::size_t>(dims_[m]);
    }
    return o;
  }

 private:
  static std::size_t count(const std::vector<int>& d) {
    if (d.empty()) return 0;
    std::size_t n = 1;
    for (int x : d) {
      if (x <= 0) throw dimension_error("Tensor: dimensions must be positive");
      n *= static_cast<std::size_t>(x);
    }
    return n;
  }
  std::vector<int> dims_;
  std::vector<T> v_;
};

// Y = X x_mode A on the GPU (FP64 DMMA).  A is r x n_mode.
inline Tensor<double> mode_multiply(const Tensor<double>& x, const Matrix<double>& a, int mode) {
  if (mode < 0 || mode >= x.order()) throw dimension_error("mode_multiply: mode out of range");
  if (a.cols() != x.dim(mode))
    throw dimension_error("mode_multiply: A has " + std::to_string(a.cols()) +
                          " columns, mode extent is " + std::to_string(x.dim(mode)));
  if (a.rows() <= 0) throw dimension_error("mode_multiply: A must have positive row count");
  std::vector<int> yd = x.dims();
  yd[mode] = a.rows();
  Tensor<double> y(yd);
  gpu::check(tsg_mode_multiply(gpu::context(), x.order(), x.dims().data(), x.data(), a.rows(),
                               a.data(), mode, y.data(), nullptr),
             "mode_multiply");
  return y;
}

// T = Complex: the complex DMMA GEMM (tsg_zmode_multiply, csrc/zsolve.cu).
inline Tensor<Complex> mode_multiply(const Tensor<Complex>& x, const Matrix<Complex>& a, int mode) {
  if (mode < 0 || mode >= x.order()) throw dimension_error("mode_multiply: mode out of range");
  if (a.cols() != x.dim(mode))
    throw dimension_error("mode_multiply: A has " + std::to_string(a.cols()) +
                          " columns, mode extent is " + std::to_string(x.dim(mode)));
  if (a.rows() <= 0) throw dimension_error("mode_multiply: A must have positive row count");
  std::vector<int> yd = x.dims();
  yd[mode] = a.rows();
  Tensor<Complex> y(yd);
  gpu::check(tsg_zmode_multiply(gpu::context(), x.order(), x.dims().data(),
                                reinterpret_cast<const double*>(x.data()), a.rows(),
                                reinterpret_cast<const double*>(a.data()), mode,
                                reinterpret_cast<double*>(y.data()), nullptr),
             "mode_multiply");
  return y;
}

}  // namespace tsylv
