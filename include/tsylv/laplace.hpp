// tsylv drop-in (B200 build) — Laplace-like solver entry points.
//
//   solve_laplace(p, cfg)              reference laplace.hpp:324-344
//   laplace_recursive(T, Bt, n_min)    reference laplace.hpp:185-195
//   laplace_merged(T, Bt, n_min)       reference laplace.hpp:202-244
//
// solve_laplace keeps the reference pipeline: host Schur
// of every coefficient (shared setup, dgees), the host solvability screen
// (singular_error with witness), then ONE call into the GPU library that runs
// forward transforms, the reduced quasi-triangular dataflow solve and the
// back transforms on the device (tsg_laplace_solve), and finally the device
// residual.  Arithmetic is real quasi-triangular throughout; the solution is
// the unique one the reference's complex default also returns (parity on X).
#pragma once
#include <stdexcept>
#include <string>
#include <vector>

#include "tsylv/config.hpp"
#include "tsylv/gpu.hpp"
#include "tsylv/lapack.hpp"
#include "tsylv/matrix.hpp"
#include "tsylv/problems.hpp"
#include "tsylv/solvability.hpp"
#include "tsylv/sylvester.hpp"
#include "tsylv/tensor.hpp"

namespace tsylv {

namespace detail {

inline void check_config(const SolverConfig& cfg, const char* who) {
  if (cfg.strategy == Strategy::merge && cfg.arithmetic == Arithmetic::real_quasitriangular)
    throw std::invalid_argument(std::string(who) +
                                ": the merge strategy needs strictly triangular (complex Schur) "
                                "coefficients; real quasi-triangular arithmetic cannot merge");
}

inline tsg_opts gpu_opts(int n_min_user) {
  tsg_opts o;
  tsg_default_opts(&o);
  o.n_min = n_min_user;  // 0: kernel-tuned tile extents
  return o;
}

inline void fill_gpu(GpuTimings& g, const tsg_report& r) {
  g.fwd_ms = r.t_fwd_ms;
  g.solve_ms = r.t_solve_ms;
  g.back_ms = r.t_back_ms;
  g.h2d_ms = r.t_h2d_ms;
  g.d2h_ms = r.t_d2h_ms;
  g.total_ms = r.t_total_ms;
  g.flops_alg = r.flops_alg;
  g.flops_exec = r.flops_exec;
}

template <typename T>
void require_reduced(const std::vector<Matrix<T>>& t, const Tensor<T>& b, int n_min,
                     const char* who, bool strict_triangular = false) {
  if (n_min < 1) throw dimension_error(std::string(who) + ": n_min must be >= 1");
  if (t.empty() || b.order() != static_cast<int>(t.size()))
    throw dimension_error(std::string(who) + ": rhs order does not match coefficient count");
  for (size_t m = 0; m < t.size(); ++m) {
    if (t[m].rows() != t[m].cols() || t[m].rows() != b.dim(static_cast<int>(m)))
      throw dimension_error(std::string(who) + ": coefficient " + std::to_string(m) +
                            " does not match rhs");
    if (strict_triangular ? !is_upper_triangular(t[m]) : !is_upper_quasi_triangular(t[m]))
      throw dimension_error(std::string(who) + ": coefficient " + std::to_string(m) +
                            (strict_triangular ? " must be upper triangular"
                                               : " must be upper quasi-triangular"));
  }
}

// solve_laplace / solve_gsylv on complex data: merge + real arithmetic is
// rejected first, then real arithmetic on complex data (laplace.hpp:304-315).
inline void check_config_complex(const SolverConfig& cfg, const char* who) {
  check_config(cfg, who);
  if (cfg.arithmetic == Arithmetic::real_quasitriangular)
    throw std::invalid_argument(std::string(who) + ": real arithmetic requires real data");
}

inline const double* dp(const Complex* p) { return reinterpret_cast<const double*>(p); }
inline double* dp(Complex* p) { return reinterpret_cast<double*>(p); }
inline std::vector<const double*> zptrs(const std::vector<Matrix<Complex>>& v) {
  std::vector<const double*> r;
  for (const auto& m : v) r.push_back(dp(m.data()));
  return r;
}
inline bool all_triangular(const std::vector<Matrix<Complex>>& v) {
  for (const auto& m : v)
    if (!is_upper_triangular(m)) return false;
  return true;
}

}  // namespace detail

inline double residual(const LaplaceProblem<double>& p, const Tensor<double>& x) {
  validate(p);
  if (x.dims() != p.rhs.dims()) throw dimension_error("residual: solution shape mismatch");
  std::vector<const double*> a;
  for (const auto& m : p.coeffs) a.push_back(m.data());
  double r = 0;
  gpu::check(tsg_residual(gpu::context(), 0, p.order(), p.rhs.dims().data(), a.data(), nullptr,
                          p.rhs.data(), x.data(), 0, &r),
             "residual");
  return r;
}

// Reduced form: sum_m X x_m T_m = Bt with upper quasi-triangular T_m.
inline Tensor<double> laplace_recursive(const std::vector<Matrix<double>>& t, Tensor<double> b,
                                        int n_min) {
  detail::require_reduced(t, b, n_min, "laplace_recursive");
  std::vector<const double*> tp;
  for (const auto& m : t) tp.push_back(m.data());
  tsg_opts o = detail::gpu_opts(n_min);
  Tensor<double> x(b.dims());
  gpu::check(tsg_laplace_reduced(gpu::context(), b.order(), b.dims().data(), tp.data(), b.data(),
                                 x.data(), &o, nullptr),
             "laplace_recursive");
  return x;
}

// Reduced form with mode merging (laplace.hpp:202-244): the reference fuses
// modes 0 and 1 while n_0 n_1 <= n_min^2 and recurses down to order-2
// solve_sylvester_tri leaves; it requires strictly upper triangular
// coefficients (complex Schur forms; for real T a real-spectrum Schur form).
// Same contract here.  On the GPU the multi-mode tiles of the dataflow solve
// play the role of the merged modes, so merging is a tile
// shape, not a dense Kronecker-sum matrix; n_min is the reference's merge
// cutoff and the GPU picks its own tile extents.  Every eigenvalue tuple is
// screened first (the reference screens each leaf with solve_sylvester_tri's
// tolerance): singular operators raise singular_error.  d = 2 forwards to
// solve_sylvester_tri(T_0, T_1, B, min(n_min, 8)) exactly as the reference.
inline Tensor<double> laplace_merged(std::vector<Matrix<double>> t, Tensor<double> b, int n_min) {
  detail::require_reduced(t, b, n_min, "laplace_merged", true);
  const int d = static_cast<int>(t.size());
  if (d == 2) {
    Matrix<double> bm(b.dim(0), b.dim(1), std::vector<double>(b.data(), b.data() + b.size()));
    Matrix<double> x = solve_sylvester_tri(t[0], t[1], std::move(bm),
                                           std::min(n_min, matrix_floor_n_min));
    return Tensor<double>(b.dims(), std::vector<double>(x.data(), x.data() + x.size()));
  }
  const Solvability s = screen_laplace_gpu(t);
  if (!s.solvable)
    throw singular_error(detail::witness_message("laplace_merged", s), s.witness,
                         s.witness_values, s.min_abs);
  std::vector<const double*> tp;
  for (const auto& m : t) tp.push_back(m.data());
  tsg_opts o = detail::gpu_opts(0);
  Tensor<double> x(b.dims());
  gpu::check(tsg_laplace_reduced(gpu::context(), d, b.dims().data(), tp.data(), b.data(),
                                 x.data(), &o, nullptr),
             "laplace_merged");
  return x;
}

inline SolveReport<double> solve_laplace(const LaplaceProblem<double>& p,
                                         const SolverConfig& cfg = {}) {
  validate(p);
  detail::check_config(cfg, "solve_laplace");
  const int d = p.order();
  SolveReport<double> rep;
  rep.n_min = cfg.n_min > 0 ? cfg.n_min : default_n_min(Family::laplace, d, cfg.strategy);
  rep.strategy = cfg.strategy;

  StopWatch sw;
  std::vector<SchurFactorization<double>> f;
  for (const auto& a : p.coeffs) f.push_back(schur(a));
  rep.timings.reduction_s = sw.lap();

  std::vector<Matrix<double>> t;
  for (const auto& s : f) t.push_back(s.t);
  const Solvability s = screen_laplace_gpu(t, cfg.singularity_tol);
  if (!s.solvable)
    throw singular_error(detail::witness_message("solve_laplace", s), s.witness, s.witness_values,
                         s.min_abs);

  std::vector<const double*> tp, up;
  for (const auto& x : f) {
    tp.push_back(x.t.data());
    up.push_back(x.u.data());
  }
  tsg_opts o = detail::gpu_opts(cfg.n_min);
  tsg_report r{};
  Tensor<double> x(p.rhs.dims());
  gpu::check(tsg_laplace_solve(gpu::context(), d, p.rhs.dims().data(), tp.data(), up.data(),
                               p.rhs.data(), x.data(), &o, &r),
             "solve_laplace");
  const double gpu_s = sw.lap();
  const double back_frac = r.t_total_ms > 0 ? (r.t_back_ms + r.t_d2h_ms) / r.t_total_ms : 0.0;
  rep.timings.back_transform_s = gpu_s * back_frac;
  rep.timings.recursion_s = gpu_s - rep.timings.back_transform_s;
  detail::fill_gpu(rep.gpu, r);
  rep.solution = std::move(x);
  rep.residual = residual(p, rep.solution);
  return rep;
}

// ---- T = Complex: complex Schur (zgees) on the host,
// the complex GPU path (tsg_zlaplace_*, csrc/zsolve.cu, csrc/zplan.cpp):
// complex DMMA transforms and the eigen-decoupled triangular fibre solve
// (wavefront back substitution for ill-conditioned eigenbases).

inline double residual(const LaplaceProblem<Complex>& p, const Tensor<Complex>& x) {
  validate(p);
  if (x.dims() != p.rhs.dims()) throw dimension_error("residual: solution shape mismatch");
  const std::vector<const double*> a = detail::zptrs(p.coeffs);
  double r = 0;
  gpu::check(tsg_zresidual(gpu::context(), 0, p.order(), p.rhs.dims().data(), a.data(), nullptr,
                           detail::dp(p.rhs.data()), detail::dp(x.data()), 0, &r),
             "residual");
  return r;
}

// Reduced form (laplace.hpp:185-195 with T = Complex).  Complex quasi-
// triangular coefficients (2x2 diagonal blocks) are accepted like the
// reference; they are first brought to triangular form by a complex Schur
// decomposition and solved through the full pipeline.
inline Tensor<Complex> laplace_recursive(const std::vector<Matrix<Complex>>& t,
                                         Tensor<Complex> b, int n_min) {
  detail::require_reduced(t, b, n_min, "laplace_recursive");
  tsg_opts o = detail::gpu_opts(n_min);
  Tensor<Complex> x(b.dims());
  if (detail::all_triangular(t)) {
    const std::vector<const double*> tp = detail::zptrs(t);
    gpu::check(tsg_zlaplace_reduced(gpu::context(), b.order(), b.dims().data(), tp.data(),
                                    detail::dp(b.data()), detail::dp(x.data()), &o, nullptr),
               "laplace_recursive");
    return x;
  }
  std::vector<SchurFactorization<Complex>> f;
  for (const auto& m : t) f.push_back(schur(m));
  std::vector<const double*> tp, up;
  for (const auto& s : f) {
    tp.push_back(detail::dp(s.t.data()));
    up.push_back(detail::dp(s.u.data()));
  }
  gpu::check(tsg_zlaplace_solve(gpu::context(), b.order(), b.dims().data(), tp.data(), up.data(),
                                detail::dp(b.data()), detail::dp(x.data()), &o, nullptr),
             "laplace_recursive");
  return x;
}

// laplace.hpp:202-244 with T = Complex: strictly triangular coefficients;
// d = 2 forwards to solve_sylvester_tri(T_0, conj(T_1), B, min(n_min, 8)).
inline Tensor<Complex> laplace_merged(std::vector<Matrix<Complex>> t, Tensor<Complex> b,
                                      int n_min) {
  detail::require_reduced(t, b, n_min, "laplace_merged", true);
  const int d = static_cast<int>(t.size());
  if (d == 2) {
    Matrix<Complex> bm(b.dim(0), b.dim(1), std::vector<Complex>(b.data(), b.data() + b.size()));
    Matrix<Complex> x = solve_sylvester_tri(t[0], conjugated(t[1]), std::move(bm),
                                            std::min(n_min, matrix_floor_n_min));
    return Tensor<Complex>(b.dims(), std::vector<Complex>(x.data(), x.data() + x.size()));
  }
  const Solvability s = check_solvable_laplace(t);
  if (!s.solvable)
    throw singular_error(detail::witness_message("laplace_merged", s), s.witness,
                         s.witness_values, s.min_abs);
  const std::vector<const double*> tp = detail::zptrs(t);
  tsg_opts o = detail::gpu_opts(0);
  Tensor<Complex> x(b.dims());
  gpu::check(tsg_zlaplace_reduced(gpu::context(), d, b.dims().data(), tp.data(),
                                  detail::dp(b.data()), detail::dp(x.data()), &o, nullptr),
             "laplace_merged");
  return x;
}

// laplace.hpp:324-344 with T = Complex (laplace_pipeline<Complex>).
inline SolveReport<Complex> solve_laplace(const LaplaceProblem<Complex>& p,
                                          const SolverConfig& cfg = {}) {
  validate(p);
  detail::check_config_complex(cfg, "solve_laplace");
  const int d = p.order();
  SolveReport<Complex> rep;
  rep.n_min = cfg.n_min > 0 ? cfg.n_min : default_n_min(Family::laplace, d, cfg.strategy);
  rep.strategy = cfg.strategy;

  StopWatch sw;
  std::vector<SchurFactorization<Complex>> f;
  for (const auto& a : p.coeffs) f.push_back(schur(a));
  rep.timings.reduction_s = sw.lap();

  std::vector<Matrix<Complex>> t;
  for (const auto& s : f) t.push_back(s.t);
  const Solvability s = check_solvable_laplace(t, cfg.singularity_tol);
  if (!s.solvable)
    throw singular_error(detail::witness_message("solve_laplace", s), s.witness, s.witness_values,
                         s.min_abs);

  std::vector<const double*> tp, up;
  for (const auto& x : f) {
    tp.push_back(detail::dp(x.t.data()));
    up.push_back(detail::dp(x.u.data()));
  }
  tsg_opts o = detail::gpu_opts(cfg.n_min);
  tsg_report r{};
  Tensor<Complex> x(p.rhs.dims());
  gpu::check(tsg_zlaplace_solve(gpu::context(), d, p.rhs.dims().data(), tp.data(), up.data(),
                                detail::dp(p.rhs.data()), detail::dp(x.data()), &o, &r),
             "solve_laplace");
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
