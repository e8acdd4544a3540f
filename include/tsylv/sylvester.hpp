// tsylv drop-in (B200 build) — the two-sided matrix solvers.
//
//   solve_sylvester_tri(A1, A2, B, n_min)     reference sylvester.hpp:194-215
//       A1 X + X A2^H = B
//   solve_gsylv_tri(A1, C, A2, B, n_min)      reference sylvester.hpp:219-241
//       A1 X + C X A2^H = B
//
// Same validation (sylv2_validate, sylvester.hpp:160-187: n_min >= 1, square
// coefficients, rhs shape, non-empty, (quasi-)triangular structure with C
// strictly upper triangular) and the same eigenvalue screen with the
// reference tolerance u (||A1||_F + ||A2||_F) (pencil form for the gsylv
// variant) before the device solve.  In real arithmetic A2^H = A2^T, so the
// first equation is the order-2 Laplace reduced form sum_m X x_m T_m = B with
// (T_0, T_1) = (A1, A2) and the second the order-2 gsylv reduced form
// X x_0 S + X x_0 Tc x_1 A_1 = B with (S, Tc, A_1) = (A1, C, A2): both run the
// reduced dataflow solve on the GPU (tsg_laplace_reduced /
// tsg_gsylv_reduced).  n_min is the reference's base-block bound; the GPU
// tiles a d = 2 problem with its own tuned extents (n_min only bounds them).
#pragma once
#include <string>
#include <vector>

#include "tsylv/config.hpp"
#include "tsylv/gpu.hpp"
#include "tsylv/matrix.hpp"
#include "tsylv/solvability.hpp"
#include "tsylv/tensor.hpp"

namespace tsylv {

namespace detail {

template <typename T>
void sylv2_validate(const Matrix<T>& a1, const Matrix<T>* c, const Matrix<T>& a2,
                    const Matrix<T>& b, int n_min, const char* who) {
  if (n_min < 1) throw dimension_error(std::string(who) + ": n_min must be >= 1");
  if (a1.rows() != a1.cols() || a2.rows() != a2.cols())
    throw dimension_error(std::string(who) + ": coefficients must be square");
  if (b.rows() != a1.rows() || b.cols() != a2.rows())
    throw dimension_error(std::string(who) + ": rhs is " + std::to_string(b.rows()) + "x" +
                          std::to_string(b.cols()) + ", expected " + std::to_string(a1.rows()) +
                          "x" + std::to_string(a2.rows()));
  if (b.rows() == 0 || b.cols() == 0) throw dimension_error(std::string(who) + ": empty system");
  // real T: quasi-triangular A1, A2 are allowed; complex T: triangular only;
  // C must be triangular
  const bool quasi_ok = !is_complex_v<T>;
  if (!is_upper_triangular(a1) && !(quasi_ok && is_upper_quasi_triangular(a1)))
    throw dimension_error(std::string(who) + (quasi_ok ? ": A1 must be upper quasi-triangular"
                                                       : ": A1 must be upper triangular"));
  if (!is_upper_triangular(a2) && !(quasi_ok && is_upper_quasi_triangular(a2)))
    throw dimension_error(std::string(who) + (quasi_ok ? ": A2 must be upper quasi-triangular"
                                                       : ": A2 must be upper triangular"));
  if (c && !is_upper_triangular(*c))
    throw dimension_error(std::string(who) + ": C must be upper triangular");
}

inline tsg_opts sylv2_opts() {
  tsg_opts o;
  tsg_default_opts(&o);
  return o;
}

}  // namespace detail

inline Matrix<double> solve_sylvester_tri(const Matrix<double>& a1, const Matrix<double>& a2,
                                          Matrix<double> b, int n_min = 32) {
  detail::sylv2_validate(a1, static_cast<const Matrix<double>*>(nullptr), a2, b, n_min,
                         "solve_sylvester_tri");
  std::vector<EigList> eigs{quasi_tri_eigenvalues(a1), quasi_tri_eigenvalues(a2)};
  for (auto& v : eigs[1]) v = std::conj(v);
  const double tol = unit_roundoff<double> * (a1.frobenius_norm() + a2.frobenius_norm());
  Solvability s = detail::min_kron_sum(eigs);
  if (s.min_abs <= tol)
    throw singular_error(detail::witness_message("solve_sylvester_tri", s), s.witness,
                         s.witness_values, s.min_abs);
  const int dims[2] = {b.rows(), b.cols()};
  const double* tp[2] = {a1.data(), a2.data()};
  tsg_opts o = detail::sylv2_opts();
  Matrix<double> x(b.rows(), b.cols());
  gpu::check(tsg_laplace_reduced(gpu::context(), 2, dims, tp, b.data(), x.data(), &o, nullptr),
             "solve_sylvester_tri");
  return x;
}

inline Matrix<double> solve_gsylv_tri(const Matrix<double>& a1, const Matrix<double>& c,
                                      const Matrix<double>& a2, Matrix<double> b,
                                      int n_min = 32) {
  detail::sylv2_validate(a1, &c, a2, b, n_min, "solve_gsylv_tri");
  if (c.rows() != a1.rows()) throw dimension_error("solve_gsylv_tri: C must match A1");
  std::vector<EigList> tail{quasi_tri_eigenvalues(a2)};
  for (auto& v : tail[0]) v = std::conj(v);
  const double tol = unit_roundoff<double> *
                     (a1.frobenius_norm() + c.frobenius_norm() + a2.frobenius_norm());
  Solvability s = detail::min_pencil_product(a1, c, tail);
  if (s.min_abs <= tol)
    throw singular_error(detail::witness_message("solve_gsylv_tri", s), s.witness,
                         s.witness_values, s.min_abs);
  const int dims[2] = {b.rows(), b.cols()};
  const double* tail_p[1] = {a2.data()};
  tsg_opts o = detail::sylv2_opts();
  Matrix<double> x(b.rows(), b.cols());
  gpu::check(tsg_gsylv_reduced(gpu::context(), 2, dims, a1.data(), c.data(), tail_p, b.data(),
                               x.data(), &o, nullptr),
             "solve_gsylv_tri");
  return x;
}

// ---- T = Complex: A1 X + X A2^H = B is the order-2 Laplace reduced form with
// (T_0, T_1) = (A1, conj(A2)); A1 X + C X A2^H = B the order-2 gsylv reduced
// form with (S, Tc, A_1) = (A1, C, conj(A2)) (tsg_zlaplace_reduced /
// tsg_zgsylv_reduced).  Same validation and eigenvalue screens.
inline Matrix<Complex> solve_sylvester_tri(const Matrix<Complex>& a1, const Matrix<Complex>& a2,
                                           Matrix<Complex> b, int n_min = 32) {
  detail::sylv2_validate(a1, static_cast<const Matrix<Complex>*>(nullptr), a2, b, n_min,
                         "solve_sylvester_tri");
  std::vector<EigList> eigs{quasi_tri_eigenvalues(a1), quasi_tri_eigenvalues(a2)};
  for (auto& v : eigs[1]) v = std::conj(v);
  const double tol = unit_roundoff<double> * (a1.frobenius_norm() + a2.frobenius_norm());
  Solvability s = detail::min_kron_sum(eigs);
  if (s.min_abs <= tol)
    throw singular_error(detail::witness_message("solve_sylvester_tri", s), s.witness,
                         s.witness_values, s.min_abs);
  const int dims[2] = {b.rows(), b.cols()};
  const Matrix<Complex> a2c = conjugated(a2);
  const double* tp[2] = {reinterpret_cast<const double*>(a1.data()),
                         reinterpret_cast<const double*>(a2c.data())};
  tsg_opts o = detail::sylv2_opts();
  Matrix<Complex> x(b.rows(), b.cols());
  gpu::check(tsg_zlaplace_reduced(gpu::context(), 2, dims, tp,
                                  reinterpret_cast<const double*>(b.data()),
                                  reinterpret_cast<double*>(x.data()), &o, nullptr),
             "solve_sylvester_tri");
  return x;
}

inline Matrix<Complex> solve_gsylv_tri(const Matrix<Complex>& a1, const Matrix<Complex>& c,
                                       const Matrix<Complex>& a2, Matrix<Complex> b,
                                       int n_min = 32) {
  detail::sylv2_validate(a1, &c, a2, b, n_min, "solve_gsylv_tri");
  if (c.rows() != a1.rows()) throw dimension_error("solve_gsylv_tri: C must match A1");
  std::vector<EigList> tail{quasi_tri_eigenvalues(a2)};
  for (auto& v : tail[0]) v = std::conj(v);
  const double tol = unit_roundoff<double> *
                     (a1.frobenius_norm() + c.frobenius_norm() + a2.frobenius_norm());
  Solvability s = detail::min_pencil_product(a1, c, tail);
  if (s.min_abs <= tol)
    throw singular_error(detail::witness_message("solve_gsylv_tri", s), s.witness,
                         s.witness_values, s.min_abs);
  const int dims[2] = {b.rows(), b.cols()};
  const Matrix<Complex> a2c = conjugated(a2);
  const double* tail_p[1] = {reinterpret_cast<const double*>(a2c.data())};
  tsg_opts o = detail::sylv2_opts();
  Matrix<Complex> x(b.rows(), b.cols());
  gpu::check(tsg_zgsylv_reduced(gpu::context(), 2, dims, reinterpret_cast<const double*>(a1.data()),
                                reinterpret_cast<const double*>(c.data()), tail_p,
                                reinterpret_cast<const double*>(b.data()),
                                reinterpret_cast<double*>(x.data()), &o, nullptr),
             "solve_gsylv_tri");
  return x;
}

}  // namespace tsylv
