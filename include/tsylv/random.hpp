// tsylv drop-in (B200 build) — deterministic inputs shared by the GPU path
// and the oracle.  RandomStream restates the reference's published stream
// (random.hpp:16-62): std::mt19937_64, uniform = (x >> 11) * 2^-53, and a
// Box-Muller normal with the sine member cached; matrices and tensors are
// filled in storage (column-major) order.  tests/test_abi.py
// (test_random_stream_bit_exact, test_make_problem_bit_exact) pins it
// bit-for-bit against the reference build in oracle/_ref.
//
// The BASELINE.json configurations are generated here (draw order:
// coefficients in mode order, then the right-hand side):
//   kind 1  convection-diffusion  A = (n+1)^2 tridiag(-1,2,-1) + c (n+1)/2 tridiag(-1,0,1),
//           c ~ U(0.5, 2) per mode                              (config C1)
//   kind 2  A = G/sqrt(n) + 3 I, G iid N(0,1)                   (configs C2, C3, C4)
//   kind 5  gsylv A X + B X (C x ... x C) = D with A = G_A/sqrt(n0) + 4 I,
//           B = G_B/sqrt(n0), C = G_C/(2 sqrt(nc)), posed as coeffs
//           {A, C^T, ..., C^T}, c = B                          (config C5)
#pragma once
#include <cmath>
#include <cstdint>
#include <numbers>
#include <random>
#include <vector>

#include "tsylv/matrix.hpp"
#include "tsylv/problems.hpp"
#include "tsylv/scalar.hpp"
#include "tsylv/tensor.hpp"

namespace tsylv {

class RandomStream {
 public:
  explicit RandomStream(std::uint64_t seed) : mt_(seed) {}
  double uniform() { return static_cast<double>(mt_() >> 11) * 0x1.0p-53; }
  double normal() {
    if (cached_) {
      cached_ = false;
      return sin_member_;
    }
    const double a = 1.0 - uniform();
    const double b = uniform();
    const double rad = std::sqrt(-2.0 * std::log(a));
    const double ang = 2.0 * std::numbers::pi * b;
    sin_member_ = rad * std::sin(ang);
    cached_ = true;
    return rad * std::cos(ang);
  }
  // Standard normal scalar of type T; complex draws have unit total variance
  // (random.hpp:50-57).  The reference builds T(normal() * .., normal() * ..)
  // in one constructor call, whose argument evaluation order is unspecified;
  // g++ (the toolchain of its CMake build and of oracle/_ref) evaluates the
  // imaginary argument first, so the stream is consumed imaginary part first
  // (pinned by tests/test_gpu_complex.py::test_zgenerators_bit_exact).
  template <typename T>
  T draw() {
    if constexpr (is_complex_v<T>) {
      const double im = normal() * std::numbers::sqrt2 / 2.0;
      const double re = normal() * std::numbers::sqrt2 / 2.0;
      return T(re, im);
    } else {
      return static_cast<T>(normal());
    }
  }

 private:
  std::mt19937_64 mt_;
  double sin_member_ = 0;
  bool cached_ = false;
};

inline Matrix<double> randn_matrix(RandomStream& r, int rows, int cols) {
  Matrix<double> m(rows, cols);
  for (std::size_t i = 0; i < m.size(); ++i) m.data()[i] = r.normal();
  return m;
}
inline Tensor<double> randn_tensor(RandomStream& r, const std::vector<int>& dims) {
  Tensor<double> t(dims);
  for (std::size_t i = 0; i < t.size(); ++i) t.data()[i] = r.normal();
  return t;
}

// Elementwise m / s (division, as BASELINE.json writes G/sqrt(n)).
inline void divide(Matrix<double>& m, double s) {
  for (std::size_t i = 0; i < m.size(); ++i) m.data()[i] /= s;
}

inline Matrix<double> convection_diffusion(int n, double c) {
  const double h2 = static_cast<double>(n + 1) * (n + 1), h1 = c * (n + 1) / 2.0;
  Matrix<double> a(n, n);
  for (int i = 0; i < n; ++i) {
    a(i, i) = 2.0 * h2;
    if (i + 1 < n) {
      a(i, i + 1) = -h2 + h1;  // super-diagonal
      a(i + 1, i) = -h2 - h1;  // sub-diagonal
    }
  }
  return a;
}

inline LaplaceProblem<double> baseline_laplace(int kind, const std::vector<int>& dims,
                                               std::uint64_t seed) {
  RandomStream r(seed);
  LaplaceProblem<double> p;
  for (int n : dims) {
    if (kind == 1) {
      p.coeffs.push_back(convection_diffusion(n, 0.5 + 1.5 * r.uniform()));
    } else {
      Matrix<double> g = randn_matrix(r, n, n);
      divide(g, std::sqrt(static_cast<double>(n)));
      for (int i = 0; i < n; ++i) g(i, i) += 3.0;
      p.coeffs.push_back(std::move(g));
    }
  }
  p.rhs = randn_tensor(r, dims);
  return p;
}

inline GSylvProblem<double> baseline_gsylv(const std::vector<int>& dims, std::uint64_t seed) {
  RandomStream r(seed);
  const int n0 = dims[0], nc = dims[1];
  Matrix<double> a = randn_matrix(r, n0, n0);
  Matrix<double> b = randn_matrix(r, n0, n0);
  Matrix<double> c = randn_matrix(r, nc, nc);
  divide(a, std::sqrt(static_cast<double>(n0)));
  for (int i = 0; i < n0; ++i) a(i, i) += 4.0;
  divide(b, std::sqrt(static_cast<double>(n0)));
  divide(c, 2.0 * std::sqrt(static_cast<double>(nc)));
  GSylvProblem<double> p;
  p.coeffs.push_back(std::move(a));
  const Matrix<double> ct = transposed(c);
  for (std::size_t m = 1; m < dims.size(); ++m) p.coeffs.push_back(ct);
  p.c = std::move(b);
  p.rhs = randn_tensor(r, dims);
  return p;
}

// ---- reduced-form (triangular) instances, real arithmetic ----------------
// The reference's correctness-suite generators (random.hpp:79-223) for
// T = double, drawing in the same order: strictly-upper Gaussian entries
// column by column, then the diagonal.

// Upper triangular, Gaussian entries, diagonal |N(0,1)| + floor_re.
inline Matrix<double> randn_triangular_posdiag(RandomStream& rng, int n, double floor_re = 1.0) {
  Matrix<double> m(n, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= j; ++i) m(i, j) = rng.normal();
  for (int i = 0; i < n; ++i) m(i, i) = std::abs(rng.normal()) + floor_re;
  return m;
}

// Upper triangular, diagonal magnitudes in [lo, hi] with a random sign.
inline Matrix<double> randn_triangular_ringdiag(RandomStream& rng, int n, double lo, double hi) {
  Matrix<double> m(n, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= j; ++i) m(i, j) = rng.normal();
  for (int i = 0; i < n; ++i) {
    const double r = lo + (hi - lo) * rng.uniform();
    m(i, i) = rng.uniform() < 0.5 ? -r : r;
  }
  return m;
}

// Laplace: diagonals >= 1, so every eigenvalue sum is >= d.
inline LaplaceProblem<double> random_reduced_laplace(RandomStream& rng, const std::vector<int>& dims) {
  LaplaceProblem<double> p;
  for (int n : dims) p.coeffs.push_back(randn_triangular_posdiag(rng, n, 1.0));
  p.rhs = randn_tensor(rng, dims);
  return p;
}

// gsylv: a0_ii >= 1, |c_ii| <= 0.09, |prod of later diagonals| <= 0.9.
inline GSylvProblem<double> random_reduced_gsylv(RandomStream& rng, const std::vector<int>& dims) {
  GSylvProblem<double> p;
  const int n0 = dims[0];
  p.coeffs.push_back(randn_triangular_posdiag(rng, n0, 1.0));
  p.c = randn_triangular_ringdiag(rng, n0, 0.05, 0.3);
  p.c *= 0.3;
  for (std::size_t m = 1; m < dims.size(); ++m) p.coeffs.push_back(randn_triangular_ringdiag(rng, dims[m], 0.3, 0.95));
  p.rhs = randn_tensor(rng, dims);
  return p;
}

// ---- typed generators (random.hpp:64-223 for any T; T = Complex is the
// reference's complex correctness suite).  Same draw
// order as the reference: column-major fills, triangular entries i <= j
// column by column, then the diagonal.
template <typename T>
Matrix<T> randn_matrix(RandomStream& r, int rows, int cols) {
  Matrix<T> m(rows, cols);
  for (int j = 0; j < cols; ++j)
    for (int i = 0; i < rows; ++i) m(i, j) = r.draw<T>();
  return m;
}
template <typename T>
Tensor<T> randn_tensor(RandomStream& r, const std::vector<int>& dims) {
  Tensor<T> t(dims);
  for (std::size_t i = 0; i < t.size(); ++i) t.data()[i] = r.draw<T>();
  return t;
}
template <typename T>
Matrix<T> randn_triangular(RandomStream& r, int n, double diag_shift = 0) {
  Matrix<T> m(n, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= j; ++i) m(i, j) = r.draw<T>();
  for (int i = 0; i < n; ++i) m(i, i) += T(diag_shift);
  return m;
}
template <typename T>
Matrix<T> randn_triangular_posdiag(RandomStream& r, int n, double floor_re = 1.0) {
  Matrix<T> m = randn_triangular<T>(r, n, 0);
  for (int i = 0; i < n; ++i) {
    const double re = std::abs(r.normal()) + floor_re;
    if constexpr (is_complex_v<T>) {
      const double im = 0.4 * r.normal();
      m(i, i) = T(re, im);
    } else {
      m(i, i) = T(re);
    }
  }
  return m;
}
template <typename T>
Matrix<T> randn_triangular_ringdiag(RandomStream& r, int n, double lo, double hi) {
  Matrix<T> m = randn_triangular<T>(r, n, 0);
  for (int i = 0; i < n; ++i) {
    const double rad = lo + (hi - lo) * r.uniform();
    if constexpr (is_complex_v<T>) {
      const double th = 2.0 * std::numbers::pi * r.uniform();
      m(i, i) = T(rad * std::cos(th), rad * std::sin(th));
    } else {
      m(i, i) = T(r.uniform() < 0.5 ? -rad : rad);
    }
  }
  return m;
}
template <typename T>
LaplaceProblem<T> random_laplace_problem(RandomStream& r, const std::vector<int>& dims) {
  LaplaceProblem<T> p;
  for (int n : dims) {
    Matrix<T> a = randn_matrix<T>(r, n, n);
    const double shift = 1.0 + 2.0 * std::sqrt(static_cast<double>(n));
    for (int i = 0; i < n; ++i) a(i, i) += T(shift);
    p.coeffs.push_back(std::move(a));
  }
  p.rhs = randn_tensor<T>(r, dims);
  return p;
}
template <typename T>
GSylvProblem<T> random_gsylv_problem(RandomStream& r, const std::vector<int>& dims) {
  GSylvProblem<T> p;
  const int n0 = dims[0];
  {
    Matrix<T> a = randn_matrix<T>(r, n0, n0);
    const double shift = 1.0 + 2.0 * std::sqrt(static_cast<double>(n0));
    for (int i = 0; i < n0; ++i) a(i, i) += T(shift);
    p.coeffs.push_back(std::move(a));
  }
  p.c = randn_matrix<T>(r, n0, n0);
  p.c *= T(0.25 / std::sqrt(static_cast<double>(n0)));
  for (std::size_t m = 1; m < dims.size(); ++m) {
    const int n = dims[m];
    Matrix<T> a = randn_matrix<T>(r, n, n);
    a *= T(0.45 / std::sqrt(static_cast<double>(n)));
    p.coeffs.push_back(std::move(a));
  }
  p.rhs = randn_tensor<T>(r, dims);
  return p;
}
template <typename T>
LaplaceProblem<T> random_reduced_laplace(RandomStream& r, const std::vector<int>& dims) {
  LaplaceProblem<T> p;
  for (int n : dims) p.coeffs.push_back(randn_triangular_posdiag<T>(r, n, 1.0));
  p.rhs = randn_tensor<T>(r, dims);
  return p;
}
template <typename T>
GSylvProblem<T> random_reduced_gsylv(RandomStream& r, const std::vector<int>& dims) {
  GSylvProblem<T> p;
  const int n0 = dims[0];
  p.coeffs.push_back(randn_triangular_posdiag<T>(r, n0, 1.0));
  p.c = randn_triangular_ringdiag<T>(r, n0, 0.05, 0.3);
  p.c *= T(0.3);
  for (std::size_t m = 1; m < dims.size(); ++m)
    p.coeffs.push_back(randn_triangular_ringdiag<T>(r, dims[m], 0.3, 0.95));
  p.rhs = randn_tensor<T>(r, dims);
  return p;
}

}  // namespace tsylv
