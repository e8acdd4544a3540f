// tsylv drop-in (B200 build) — generalized Sylvester solver entry points.
//
//   solve_gsylv(p, cfg)                    reference gsylv.hpp:311-331
//   gsylv_recursive(T, C, Bt, n_min)       reference gsylv.hpp:149-159
//   gsylv_merged(T, C, Bt, n_min)          reference gsylv.hpp:167-232
//
// Pipeline of gsylv_pipeline (gsylv.hpp:236-302): QZ of (A_0, C) and Schur of
// every tail coefficient on the host (shared setup), the pencil screen, then
// the GPU: B~ = B x_0 Q^T x_m U_m^T, the reduced dataflow solve with the
// factored chain W_m (see csrc/solve.cu), X = X~ x_0 Z x_m U_m.
#pragma once
#include <string>
#include <vector>

#include "tsylv/laplace.hpp"

namespace tsylv {

inline double residual(const GSylvProblem<double>& p, const Tensor<double>& x) {
  validate(p);
  if (x.dims() != p.rhs.dims()) throw dimension_error("residual: solution shape mismatch");
  std::vector<const double*> a;
  for (const auto& m : p.coeffs) a.push_back(m.data());
  double r = 0;
  gpu::check(tsg_residual(gpu::context(), 1, p.order(), p.rhs.dims().data(), a.data(), p.c.data(),
                          p.rhs.data(), x.data(), 0, &r),
             "residual");
  return r;
}

inline Tensor<double> gsylv_recursive(const std::vector<Matrix<double>>& t, const Matrix<double>& c,
                                      Tensor<double> b, int n_min) {
  detail::require_reduced(t, b, n_min, "gsylv_recursive");
  if (t.size() < 2) throw dimension_error("gsylv_recursive: need at least two modes");
  if (c.rows() != t[0].rows() || c.cols() != t[0].cols())
    throw dimension_error("gsylv_recursive: C must match A_0");
  if (!is_upper_triangular(c)) throw dimension_error("gsylv_recursive: C must be upper triangular");
  std::vector<const double*> tail;
  for (size_t m = 1; m < t.size(); ++m) tail.push_back(t[m].data());
  tsg_opts o = detail::gpu_opts(n_min);
  Tensor<double> x(b.dims());
  gpu::check(tsg_gsylv_reduced(gpu::context(), b.order(), b.dims().data(), t[0].data(), c.data(),
                               tail.data(), b.data(), x.data(), &o, nullptr),
             "gsylv_recursive");
  return x;
}

// Reduced form with mode merging (gsylv.hpp:167-232): the reference fuses
// the last two modes (kron(A_{d-1}, A_{d-2})) while n_{d-2} n_{d-1} <=
// n_min^2 and recurses to order-2 solve_gsylv_tri leaves; strictly upper
// triangular coefficients and C are required (require_reduced_gsylv with
// strict = true, gsylv.hpp:130-141).  On the GPU the pencil tiles of the
// dataflow solve stand in for the merged modes; the pencil screen runs
// first.  d = 2 forwards to solve_gsylv_tri(T_0, C, T_1, B, min(n_min, 8)).
inline Tensor<double> gsylv_merged(std::vector<Matrix<double>> t, Matrix<double> c,
                                   Tensor<double> b, int n_min) {
  detail::require_reduced(t, b, n_min, "gsylv_merged", true);
  if (t.size() < 2) throw dimension_error("gsylv_merged: need at least two modes");
  if (c.rows() != t[0].rows() || c.cols() != t[0].cols())
    throw dimension_error("gsylv_merged: C must match A_0");
  if (!is_upper_triangular(c)) throw dimension_error("gsylv_merged: C must be upper triangular");
  const int d = static_cast<int>(t.size());
  if (d == 2) {
    Matrix<double> bm(b.dim(0), b.dim(1), std::vector<double>(b.data(), b.data() + b.size()));
    Matrix<double> x = solve_gsylv_tri(t[0], c, t[1], std::move(bm),
                                       std::min(n_min, matrix_floor_n_min));
    return Tensor<double>(b.dims(), std::vector<double>(x.data(), x.data() + x.size()));
  }
  const Solvability s = screen_gsylv_gpu(t, c);
  if (!s.solvable)
    throw singular_error(detail::witness_message("gsylv_merged", s), s.witness, s.witness_values,
                         s.min_abs);
  std::vector<const double*> tail;
  for (size_t m = 1; m < t.size(); ++m) tail.push_back(t[m].data());
  tsg_opts o = detail::gpu_opts(0);
  Tensor<double> x(b.dims());
  gpu::check(tsg_gsylv_reduced(gpu::context(), d, b.dims().data(), t[0].data(), c.data(),
                               tail.data(), b.data(), x.data(), &o, nullptr),
             "gsylv_merged");
  return x;
}

inline SolveReport<double> solve_gsylv(const GSylvProblem<double>& p, const SolverConfig& cfg = {}) {
  validate(p);
  detail::check_config(cfg, "solve_gsylv");
  const int d = p.order();
  SolveReport<double> rep;
  rep.n_min = cfg.n_min > 0 ? cfg.n_min : default_n_min(Family::gsylv, d, cfg.strategy);
  rep.strategy = cfg.strategy;

  StopWatch sw;
  GeneralizedSchurFactorization<double> g = qz(p.coeffs[0], p.c);
  std::vector<SchurFactorization<double>> f;
  for (int m = 1; m < d; ++m) f.push_back(schur(p.coeffs[m]));
  rep.timings.reduction_s = sw.lap();

  std::vector<Matrix<double>> red{g.s};
  for (const auto& x : f) red.push_back(x.t);
  const Solvability s = screen_gsylv_gpu(red, g.t, cfg.singularity_tol);
  if (!s.solvable)
    throw singular_error(detail::witness_message("solve_gsylv", s), s.witness, s.witness_values,
                         s.min_abs);

  std::vector<const double*> tp, up;
  for (const auto& x : f) {
    tp.push_back(x.t.data());
    up.push_back(x.u.data());
  }
  tsg_opts o = detail::gpu_opts(cfg.n_min);
  tsg_report r{};
  Tensor<double> x(p.rhs.dims());
  gpu::check(tsg_gsylv_solve(gpu::context(), d, p.rhs.dims().data(), g.s.data(), g.t.data(),
                             g.u.data(), g.z.data(), tp.data(), up.data(), p.rhs.data(), x.data(),
                             &o, &r),
             "solve_gsylv");
  const double gpu_s = sw.lap();
  const double back_frac = r.t_total_ms > 0 ? (r.t_back_ms + r.t_d2h_ms) / r.t_total_ms : 0.0;
  rep.timings.back_transform_s = gpu_s * back_frac;
  rep.timings.recursion_s = gpu_s - rep.timings.back_transform_s;
  detail::fill_gpu(rep.gpu, r);
  rep.solution = std::move(x);
  rep.residual = residual(p, rep.solution);
  return rep;
}

// ---- T = Complex: complex QZ (zgges) of (A_0, C) and
// complex Schur of the tails on the host, the complex GPU path
// (tsg_zgsylv_*): complex DMMA transforms (Q^H / Z on mode 0) and the pencil
// fibre solve (S + z Tc) x = b along mode 0 with the tails in their
// eigenbases (z = product of tail eigenvalues).

inline double residual(const GSylvProblem<Complex>& p, const Tensor<Complex>& x) {
  validate(p);
  if (x.dims() != p.rhs.dims()) throw dimension_error("residual: solution shape mismatch");
  const std::vector<const double*> a = detail::zptrs(p.coeffs);
  double r = 0;
  gpu::check(tsg_zresidual(gpu::context(), 1, p.order(), p.rhs.dims().data(), a.data(),
                           detail::dp(p.c.data()), detail::dp(p.rhs.data()), detail::dp(x.data()),
                           0, &r),
             "residual");
  return r;
}

namespace detail {
inline void require_reduced_gsylv(const std::vector<Matrix<Complex>>& t, const Matrix<Complex>& c,
                                  const Tensor<Complex>& b, int n_min, bool strict,
                                  const char* who) {
  require_reduced(t, b, n_min, who, strict);
  if (t.size() < 2) throw dimension_error(std::string(who) + ": need at least two modes");
  if (c.rows() != t[0].rows() || c.cols() != t[0].cols())
    throw dimension_error(std::string(who) + ": C must match A_0");
  if (!is_upper_triangular(c)) throw dimension_error(std::string(who) + ": C must be upper triangular");
}
// Full complex gsylv solve from a problem's coefficients (QZ + Schur here).
inline Tensor<Complex> zgsylv_full(const std::vector<Matrix<Complex>>& a, const Matrix<Complex>& c,
                                   const Tensor<Complex>& b, tsg_opts* o, tsg_report* r,
                                   const char* who) {
  const int d = static_cast<int>(a.size());
  GeneralizedSchurFactorization<Complex> g = qz(a[0], c);
  std::vector<SchurFactorization<Complex>> f;
  for (int m = 1; m < d; ++m) f.push_back(schur(a[m]));
  std::vector<const double*> tp, up;
  for (const auto& x : f) {
    tp.push_back(dp(x.t.data()));
    up.push_back(dp(x.u.data()));
  }
  Tensor<Complex> x(b.dims());
  gpu::check(tsg_zgsylv_solve(gpu::context(), d, b.dims().data(), dp(g.s.data()), dp(g.t.data()),
                              dp(g.u.data()), dp(g.z.data()), tp.data(), up.data(), dp(b.data()),
                              dp(x.data()), o, r),
             who);
  return x;
}
}  // namespace detail

// gsylv.hpp:149-159 with T = Complex; quasi-triangular complex factors go
// through a QZ / Schur reduction first (as laplace_recursive<Complex>).
inline Tensor<Complex> gsylv_recursive(const std::vector<Matrix<Complex>>& t,
                                       const Matrix<Complex>& c, Tensor<Complex> b, int n_min) {
  detail::require_reduced_gsylv(t, c, b, n_min, false, "gsylv_recursive");
  tsg_opts o = detail::gpu_opts(n_min);
  if (!detail::all_triangular(t)) return detail::zgsylv_full(t, c, b, &o, nullptr, "gsylv_recursive");
  std::vector<const double*> tail;
  for (size_t m = 1; m < t.size(); ++m) tail.push_back(detail::dp(t[m].data()));
  Tensor<Complex> x(b.dims());
  gpu::check(tsg_zgsylv_reduced(gpu::context(), b.order(), b.dims().data(), detail::dp(t[0].data()),
                                detail::dp(c.data()), tail.data(), detail::dp(b.data()),
                                detail::dp(x.data()), &o, nullptr),
             "gsylv_recursive");
  return x;
}

// gsylv.hpp:167-232 with T = Complex: strictly triangular factors; d = 2
// forwards to solve_gsylv_tri(T_0, C, conj(T_1), B, min(n_min, 8)).
inline Tensor<Complex> gsylv_merged(std::vector<Matrix<Complex>> t, Matrix<Complex> c,
                                    Tensor<Complex> b, int n_min) {
  detail::require_reduced_gsylv(t, c, b, n_min, true, "gsylv_merged");
  const int d = static_cast<int>(t.size());
  if (d == 2) {
    Matrix<Complex> bm(b.dim(0), b.dim(1), std::vector<Complex>(b.data(), b.data() + b.size()));
    Matrix<Complex> x = solve_gsylv_tri(t[0], c, conjugated(t[1]), std::move(bm),
                                        std::min(n_min, matrix_floor_n_min));
    return Tensor<Complex>(b.dims(), std::vector<Complex>(x.data(), x.data() + x.size()));
  }
  const Solvability s = check_solvable_gsylv(t, c);
  if (!s.solvable)
    throw singular_error(detail::witness_message("gsylv_merged", s), s.witness, s.witness_values,
                         s.min_abs);
  std::vector<const double*> tail;
  for (size_t m = 1; m < t.size(); ++m) tail.push_back(detail::dp(t[m].data()));
  tsg_opts o = detail::gpu_opts(0);
  Tensor<Complex> x(b.dims());
  gpu::check(tsg_zgsylv_reduced(gpu::context(), d, b.dims().data(), detail::dp(t[0].data()),
                                detail::dp(c.data()), tail.data(), detail::dp(b.data()),
                                detail::dp(x.data()), &o, nullptr),
             "gsylv_merged");
  return x;
}

// gsylv.hpp:311-331 with T = Complex (gsylv_pipeline<Complex>).
inline SolveReport<Complex> solve_gsylv(const GSylvProblem<Complex>& p, const SolverConfig& cfg = {}) {
  validate(p);
  detail::check_config_complex(cfg, "solve_gsylv");
  const int d = p.order();
  SolveReport<Complex> rep;
  rep.n_min = cfg.n_min > 0 ? cfg.n_min : default_n_min(Family::gsylv, d, cfg.strategy);
  rep.strategy = cfg.strategy;

  StopWatch sw;
  GeneralizedSchurFactorization<Complex> g = qz(p.coeffs[0], p.c);
  std::vector<SchurFactorization<Complex>> f;
  for (int m = 1; m < d; ++m) f.push_back(schur(p.coeffs[m]));
  rep.timings.reduction_s = sw.lap();

  std::vector<Matrix<Complex>> red{g.s};
  for (const auto& x : f) red.push_back(x.t);
  const Solvability s = check_solvable_gsylv(red, g.t, cfg.singularity_tol);
  if (!s.solvable)
    throw singular_error(detail::witness_message("solve_gsylv", s), s.witness, s.witness_values,
                         s.min_abs);

  std::vector<const double*> tp, up;
  for (const auto& x : f) {
    tp.push_back(detail::dp(x.t.data()));
    up.push_back(detail::dp(x.u.data()));
  }
  tsg_opts o = detail::gpu_opts(cfg.n_min);
  tsg_report r{};
  Tensor<Complex> x(p.rhs.dims());
  gpu::check(tsg_zgsylv_solve(gpu::context(), d, p.rhs.dims().data(), detail::dp(g.s.data()),
                              detail::dp(g.t.data()), detail::dp(g.u.data()), detail::dp(g.z.data()),
                              tp.data(), up.data(), detail::dp(p.rhs.data()), detail::dp(x.data()),
                              &o, &r),
             "solve_gsylv");
  const double gpu_s = sw.lap();
  const double back_frac = r.t_total_ms > 0 ? (r.t_back_ms + r.t_d2h_ms) / r.t_total_ms : 0.0;
  rep.timings.back_transform_s = gpu_s * back_frac;
  rep.timings.recursion_s = gpu_s - rep.timings.back_transform_s;
  detail::fill_gpu(rep.gpu, r);
  rep.solution = std::move(x);
  rep.residual = residual(p, rep.solution);
  return rep;
}

}  // namespace tsylv
