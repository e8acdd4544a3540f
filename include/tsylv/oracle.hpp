// tsylv drop-in (B200 build) — tsylv::oracle, the reference's validation API
// (proj/include/tsylv/oracle.hpp).
//
//   oracle::residual(p, X)                  oracle.hpp:231-268 (Laplace, gsylv)
//   oracle::solve(p, size_cap)              oracle.hpp:205-221
//   oracle::assemble_laplace_matrix(A, cap) oracle.hpp:41-71
//   oracle::assemble_gsylv_matrix(A, C, cap) oracle.hpp:75-127
//
// residual: ||op(X) - B||_F / (scale(op) ||X||_F + ||B||_F) through mode
// products only, on the device (tsg_residual; the full-size parity tests pin
// its value against the reference's oracle::residual on the same X).
// solve: the dense Kronecker operator on vec(X) (mode 0 fastest) assembled on
// the host, capped at default_size_cap unknowns like the reference, and
// solved by LU with partial pivoting (LAPACK dgetrf/dgetrs from the same
// OpenBLAS as the Schur setup); a pivot <= u ||op||_F raises singular_error
// with the column, as dense_solve does (oracle.hpp:131-200).  This is the
// reference's independent cross-check, deliberately not the GPU path.
#pragma once
#include <complex>
#include <cstddef>
#include <string>
#include <vector>

#include "tsylv/gsylv.hpp"
#include "tsylv/laplace.hpp"

extern "C" {
void dgetrf_(const int* m, const int* n, double* a, const int* lda, int* ipiv, int* info);
void dgetrs_(const char* trans, const int* n, const int* nrhs, const double* a, const int* lda,
             const int* ipiv, double* b, const int* ldb, int* info);
void zgetrf_(const int* m, const int* n, std::complex<double>* a, const int* lda, int* ipiv,
             int* info);
void zgetrs_(const char* trans, const int* n, const int* nrhs, const std::complex<double>* a,
             const int* lda, const int* ipiv, std::complex<double>* b, const int* ldb, int* info);
}

namespace tsylv::oracle {

inline constexpr std::size_t default_size_cap = 4096;

namespace detail {
inline std::size_t checked_problem_size(const std::vector<int>& dims, std::size_t size_cap,
                                        const char* who) {
  std::size_t n = 1;
  for (int d : dims) n *= static_cast<std::size_t>(d);
  if (n > size_cap)
    throw dimension_error(std::string(who) + ": operator order " + std::to_string(n) +
                          " exceeds cap " + std::to_string(size_cap));
  return n;
}

template <typename T>
std::vector<int> square_dims(const std::vector<Matrix<T>>& coeffs, const char* who) {
  if (coeffs.empty()) throw dimension_error(std::string(who) + ": no coefficients");
  std::vector<int> dims;
  for (const auto& a : coeffs) {
    if (a.rows() != a.cols() || a.rows() == 0)
      throw dimension_error(std::string(who) + ": coefficients must be square, non-empty");
    dims.push_back(a.rows());
  }
  return dims;
}
inline void getrf(int n, double* a, int* piv, int* info) { dgetrf_(&n, &n, a, &n, piv, info); }
inline void getrf(int n, std::complex<double>* a, int* piv, int* info) {
  zgetrf_(&n, &n, a, &n, piv, info);
}
inline void getrs(int n, const double* a, const int* piv, double* b, int* info) {
  const int one = 1;
  dgetrs_("N", &n, &one, a, &n, piv, b, &n, info);
}
inline void getrs(int n, const std::complex<double>* a, const int* piv, std::complex<double>* b,
                  int* info) {
  const int one = 1;
  zgetrs_("N", &n, &one, a, &n, piv, b, &n, info);
}
}  // namespace detail

// sum_m I (x) .. (x) A_m (x) .. (x) I: entry (r, c) of mode m's term is
// A_m(i, j) where r and c agree in every digit except mode m's (i, j).
template <typename T>
Matrix<T> assemble_laplace_matrix(const std::vector<Matrix<T>>& coeffs,
                                  std::size_t size_cap = default_size_cap) {
  const std::vector<int> dims = detail::square_dims(coeffs, "assemble_laplace_matrix");
  const std::size_t big = detail::checked_problem_size(dims, size_cap, "assemble_laplace_matrix");
  Matrix<T> op(static_cast<int>(big), static_cast<int>(big));
  std::size_t lo = 1;  // stride of mode m
  for (std::size_t m = 0; m < coeffs.size(); ++m) {
    const std::size_t n = static_cast<std::size_t>(dims[m]), hi = big / (lo * n);
    for (std::size_t q = 0; q < hi; ++q)
      for (std::size_t j = 0; j < n; ++j)
        for (std::size_t i = 0; i < n; ++i) {
          const T a = coeffs[m](static_cast<int>(i), static_cast<int>(j));
          if (a == T{}) continue;
          for (std::size_t p = 0; p < lo; ++p)
            op(static_cast<int>(p + lo * (i + n * q)), static_cast<int>(p + lo * (j + n * q))) += a;
        }
    lo *= n;
  }
  return op;
}

// I (x) .. (x) A_0 + A_{d-1} (x) .. (x) A_1 (x) C.
template <typename T>
Matrix<T> assemble_gsylv_matrix(const std::vector<Matrix<T>>& coeffs, const Matrix<T>& c,
                                std::size_t size_cap = default_size_cap) {
  const std::vector<int> dims = detail::square_dims(coeffs, "assemble_gsylv_matrix");
  if (c.rows() != c.cols() || c.rows() != dims[0])
    throw dimension_error("assemble_gsylv_matrix: C must be square with the order of A_0");
  const std::size_t big = detail::checked_problem_size(dims, size_cap, "assemble_gsylv_matrix");
  const int n = static_cast<int>(big), d = static_cast<int>(dims.size()), n0 = dims[0];
  Matrix<T> op(n, n);
  for (int q = 0; q < n / n0; ++q)
    for (int j = 0; j < n0; ++j)
      for (int i = 0; i < n0; ++i) op(q * n0 + i, q * n0 + j) += coeffs[0](i, j);
  std::vector<int> ri(d), ci(d);
  for (int col = 0; col < n; ++col) {
    for (int m = 0, v = col; m < d; v /= dims[m], ++m) ci[m] = v % dims[m];
    for (int row = 0; row < n; ++row) {
      for (int m = 0, v = row; m < d; v /= dims[m], ++m) ri[m] = v % dims[m];
      T v = c(ri[0], ci[0]);
      for (int m = 1; m < d && v != T{}; ++m) v *= coeffs[m](ri[m], ci[m]);
      op(row, col) += v;
    }
  }
  return op;
}

template <typename T>
std::vector<T> dense_solve(Matrix<T> a, std::vector<T> b) {
  if (a.rows() != a.cols()) throw dimension_error("dense_solve: matrix must be square");
  const int n = a.rows();
  if (static_cast<int>(b.size()) != n) throw dimension_error("dense_solve: rhs length mismatch");
  if (n == 0) return b;
  const double tiny = unit_roundoff<double> * a.frobenius_norm();
  std::vector<int> piv(n);
  int info = 0;
  detail::getrf(n, a.data(), piv.data(), &info);
  if (info < 0) throw std::invalid_argument("dense_solve: dgetrf illegal argument");
  for (int k = 0; k < n; ++k)
    if (std::abs(a(k, k)) <= tiny)
      throw singular_error("dense_solve: numerically singular at column " + std::to_string(k),
                           {k}, {std::complex<double>(a(k, k))}, std::abs(a(k, k)));
  detail::getrs(n, a.data(), piv.data(), b.data(), &info);
  return b;
}

template <typename T>
Tensor<T> solve(const LaplaceProblem<T>& p, std::size_t size_cap = default_size_cap) {
  validate(p);
  std::vector<T> x = dense_solve(assemble_laplace_matrix(p.coeffs, size_cap),
                                 std::vector<T>(p.rhs.data(), p.rhs.data() + p.rhs.size()));
  return Tensor<T>(p.rhs.dims(), std::move(x));
}

template <typename T>
Tensor<T> solve(const GSylvProblem<T>& p, std::size_t size_cap = default_size_cap) {
  validate(p);
  std::vector<T> x = dense_solve(assemble_gsylv_matrix(p.coeffs, p.c, size_cap),
                                 std::vector<T>(p.rhs.data(), p.rhs.data() + p.rhs.size()));
  return Tensor<T>(p.rhs.dims(), std::move(x));
}

// T = double and T = Complex: the device residual (tsg_residual / tsg_zresidual)
template <typename T>
double residual(const LaplaceProblem<T>& p, const Tensor<T>& x) {
  return tsylv::residual(p, x);
}
template <typename T>
double residual(const GSylvProblem<T>& p, const Tensor<T>& x) {
  return tsylv::residual(p, x);
}

}  // namespace tsylv::oracle
