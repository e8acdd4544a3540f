// Flat extern "C" facade over the C++ drop-in headers (include/tsylv/), so the
// Python host mirror (paper_1905_09539_b200/api.py) calls exactly the code a
// C++ user of the reference API gets.  Signatures mirror oracle/ref_driver.cpp
// one-for-one, so parity tests call both sides the same way.  Status codes
// are those of tsylv_gpu.h.
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "tsylv/tsylv.hpp"

using namespace tsylv;

namespace {

void set_err(char* err, int errlen, const std::string& m) {
  if (!err || errlen <= 0) return;
  std::strncpy(err, m.c_str(), static_cast<size_t>(errlen - 1));
  err[errlen - 1] = 0;
}

template <typename F>
int guarded(char* err, int errlen, F&& fn) {
  try {
    fn();
    return TSG_OK;
  } catch (const dimension_error& e) {
    set_err(err, errlen, e.what());
    return TSG_EDIM;
  } catch (const singular_error& e) {
    set_err(err, errlen, e.what());
    return TSG_ESINGULAR;
  } catch (const factorization_error& e) {
    set_err(err, errlen, e.what());
    return TSG_EFACT;
  } catch (const std::invalid_argument& e) {
    set_err(err, errlen, e.what());
    return TSG_EINVAL;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return TSG_ECUDA;
  }
}

std::vector<int> dv(int d, const int* dims) { return {dims, dims + d}; }
size_t numel(int d, const int* dims) {
  size_t n = 1;
  for (int i = 0; i < d; ++i) n *= static_cast<size_t>(dims[i]);
  return n;
}
Matrix<double> mat(int r, int c, const double* p) {
  return Matrix<double>(r, c, std::vector<double>(p, p + static_cast<size_t>(r) * c));
}
Tensor<double> ten(int d, const int* dims, const double* p) {
  return Tensor<double>(dv(d, dims), std::vector<double>(p, p + numel(d, dims)));
}
SolverConfig cfg_of(int strategy, int arithmetic, int n_min) {
  SolverConfig c;
  c.n_min = n_min;
  c.strategy = strategy == 0 ? Strategy::recursion_only : Strategy::merge;
  c.arithmetic = arithmetic == 0 ? Arithmetic::complex_triangular : Arithmetic::real_quasitriangular;
  return c;
}
// info: residual, discarded_imag, reduction_s, recursion_s, back_transform_s,
// n_min, gpu fwd/solve/back/h2d/d2h/total ms, flops_alg, flops_exec (14).
void fill_info(const SolveReport<double>& r, double* info) {
  if (!info) return;
  const double v[14] = {r.residual, r.discarded_imag, r.timings.reduction_s, r.timings.recursion_s,
                        r.timings.back_transform_s, static_cast<double>(r.n_min), r.gpu.fwd_ms,
                        r.gpu.solve_ms, r.gpu.back_ms, r.gpu.h2d_ms, r.gpu.d2h_ms, r.gpu.total_ms,
                        r.gpu.flops_alg, r.gpu.flops_exec};
  std::memcpy(info, v, sizeof(v));
}

// complex (interleaved) buffers
using Z = std::complex<double>;
const Z* zc(const double* p) { return reinterpret_cast<const Z*>(p); }
Matrix<Z> zmat(int r, int c, const double* p) {
  return Matrix<Z>(r, c, std::vector<Z>(zc(p), zc(p) + static_cast<size_t>(r) * c));
}
Tensor<Z> zten(int d, const int* dims, const double* p) {
  return Tensor<Z>(dv(d, dims), std::vector<Z>(zc(p), zc(p) + numel(d, dims)));
}
std::vector<Matrix<Z>> zmats(int d, const int* dims, const double* const* t) {
  std::vector<Matrix<Z>> v;
  for (int m = 0; m < d; ++m) v.push_back(zmat(dims[m], dims[m], t[m]));
  return v;
}
template <typename M>
void zout(const M& m, double* x) {
  std::memcpy(x, m.data(), m.size() * sizeof(Z));
}
void zfill_info(const SolveReport<Z>& r, double* info) {
  if (!info) return;
  const double v[14] = {r.residual, r.discarded_imag, r.timings.reduction_s, r.timings.recursion_s,
                        r.timings.back_transform_s, static_cast<double>(r.n_min), r.gpu.fwd_ms,
                        r.gpu.solve_ms, r.gpu.back_ms, r.gpu.h2d_ms, r.gpu.d2h_ms, r.gpu.total_ms,
                        r.gpu.flops_alg, r.gpu.flops_exec};
  std::memcpy(info, v, sizeof(v));
}

}  // namespace

extern "C" {

int tsylv_solve_laplace(int d, const int* dims, const double* const* coeffs, const double* rhs,
                        int strategy, int arithmetic, int n_min, double* x, double* info, char* err,
                        int errlen) {
  return guarded(err, errlen, [&] {
    LaplaceProblem<double> p;
    for (int m = 0; m < d; ++m) p.coeffs.push_back(mat(dims[m], dims[m], coeffs[m]));
    p.rhs = ten(d, dims, rhs);
    SolveReport<double> r = solve_laplace(p, cfg_of(strategy, arithmetic, n_min));
    std::memcpy(x, r.solution.data(), r.solution.size() * sizeof(double));
    fill_info(r, info);
  });
}

int tsylv_solve_gsylv(int d, const int* dims, const double* const* coeffs, const double* c,
                      const double* rhs, int strategy, int arithmetic, int n_min, double* x,
                      double* info, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GSylvProblem<double> p;
    for (int m = 0; m < d; ++m) p.coeffs.push_back(mat(dims[m], dims[m], coeffs[m]));
    p.c = mat(dims[0], dims[0], c);
    p.rhs = ten(d, dims, rhs);
    SolveReport<double> r = solve_gsylv(p, cfg_of(strategy, arithmetic, n_min));
    std::memcpy(x, r.solution.data(), r.solution.size() * sizeof(double));
    fill_info(r, info);
  });
}

int tsylv_laplace_recursive(int d, const int* dims, const double* const* t, const double* bt,
                            int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Matrix<double>> tt;
    for (int m = 0; m < d; ++m) tt.push_back(mat(dims[m], dims[m], t[m]));
    Tensor<double> r = laplace_recursive(tt, ten(d, dims, bt), n_min);
    std::memcpy(x, r.data(), r.size() * sizeof(double));
  });
}

int tsylv_gsylv_recursive(int d, const int* dims, const double* const* t, const double* tc,
                          const double* bt, int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Matrix<double>> tt;
    for (int m = 0; m < d; ++m) tt.push_back(mat(dims[m], dims[m], t[m]));
    Tensor<double> r = gsylv_recursive(tt, mat(dims[0], dims[0], tc), ten(d, dims, bt), n_min);
    std::memcpy(x, r.data(), r.size() * sizeof(double));
  });
}

int tsylv_laplace_merged(int d, const int* dims, const double* const* t, const double* bt,
                         int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Matrix<double>> tt;
    for (int m = 0; m < d; ++m) tt.push_back(mat(dims[m], dims[m], t[m]));
    Tensor<double> r = laplace_merged(std::move(tt), ten(d, dims, bt), n_min);
    std::memcpy(x, r.data(), r.size() * sizeof(double));
  });
}

int tsylv_gsylv_merged(int d, const int* dims, const double* const* t, const double* tc,
                       const double* bt, int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Matrix<double>> tt;
    for (int m = 0; m < d; ++m) tt.push_back(mat(dims[m], dims[m], t[m]));
    Tensor<double> r = gsylv_merged(std::move(tt), mat(dims[0], dims[0], tc), ten(d, dims, bt), n_min);
    std::memcpy(x, r.data(), r.size() * sizeof(double));
  });
}

int tsylv_solve_sylvester_tri(int r, int c, const double* a1, const double* a2, const double* b,
                              int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Matrix<double> out = solve_sylvester_tri(mat(r, r, a1), mat(c, c, a2), mat(r, c, b), n_min);
    std::memcpy(x, out.data(), out.size() * sizeof(double));
  });
}

int tsylv_solve_gsylv_tri(int r, int c, const double* a1, const double* cm, const double* a2,
                          const double* b, int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Matrix<double> out =
        solve_gsylv_tri(mat(r, r, a1), mat(r, r, cm), mat(c, c, a2), mat(r, c, b), n_min);
    std::memcpy(x, out.data(), out.size() * sizeof(double));
  });
}

int tsylv_oracle_solve_laplace(int d, const int* dims, const double* const* coeffs,
                               const double* rhs, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    LaplaceProblem<double> p;
    for (int m = 0; m < d; ++m) p.coeffs.push_back(mat(dims[m], dims[m], coeffs[m]));
    p.rhs = ten(d, dims, rhs);
    Tensor<double> r = oracle::solve(p);
    std::memcpy(x, r.data(), r.size() * sizeof(double));
  });
}

int tsylv_oracle_solve_gsylv(int d, const int* dims, const double* const* coeffs, const double* c,
                             const double* rhs, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GSylvProblem<double> p;
    for (int m = 0; m < d; ++m) p.coeffs.push_back(mat(dims[m], dims[m], coeffs[m]));
    p.c = mat(dims[0], dims[0], c);
    p.rhs = ten(d, dims, rhs);
    Tensor<double> r = oracle::solve(p);
    std::memcpy(x, r.data(), r.size() * sizeof(double));
  });
}

int tsylv_mode_multiply(int d, const int* dims, const double* xin, int r, const double* a, int mode,
                        double* y, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Tensor<double> out = mode_multiply(ten(d, dims, xin), mat(r, dims[mode], a), mode);
    std::memcpy(y, out.data(), out.size() * sizeof(double));
  });
}

int tsylv_schur(int n, const double* a, double* u, double* t, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    SchurFactorization<double> f = schur(mat(n, n, a));
    std::memcpy(u, f.u.data(), f.u.size() * sizeof(double));
    std::memcpy(t, f.t.data(), f.t.size() * sizeof(double));
  });
}

int tsylv_qz(int n, const double* a, const double* c, double* q, double* z, double* s, double* t,
             char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GeneralizedSchurFactorization<double> f = qz(mat(n, n, a), mat(n, n, c));
    std::memcpy(q, f.u.data(), f.u.size() * sizeof(double));
    std::memcpy(z, f.z.data(), f.z.size() * sizeof(double));
    std::memcpy(s, f.s.data(), f.s.size() * sizeof(double));
    std::memcpy(t, f.t.data(), f.t.size() * sizeof(double));
  });
}

double tsylv_residual_laplace(int d, const int* dims, const double* const* coeffs,
                              const double* rhs, const double* x) {
  LaplaceProblem<double> p;
  for (int m = 0; m < d; ++m) p.coeffs.push_back(mat(dims[m], dims[m], coeffs[m]));
  p.rhs = ten(d, dims, rhs);
  return oracle::residual(p, ten(d, dims, x));
}

double tsylv_residual_gsylv(int d, const int* dims, const double* const* coeffs, const double* c,
                            const double* rhs, const double* x) {
  GSylvProblem<double> p;
  for (int m = 0; m < d; ++m) p.coeffs.push_back(mat(dims[m], dims[m], coeffs[m]));
  p.c = mat(dims[0], dims[0], c);
  p.rhs = ten(d, dims, rhs);
  return oracle::residual(p, ten(d, dims, x));
}

int tsylv_check_solvable_laplace(int d, const int* dims, const double* const* t, double tol,
                                 double* min_abs, int* witness, int* solvable, char* err,
                                 int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Matrix<double>> tt;
    for (int m = 0; m < d; ++m) tt.push_back(mat(dims[m], dims[m], t[m]));
    Solvability s = check_solvable_laplace(tt, tol);
    *min_abs = s.min_abs;
    *solvable = s.solvable ? 1 : 0;
    for (size_t i = 0; i < s.witness.size(); ++i) witness[i] = s.witness[i];
  });
}

// ---- deterministic inputs (random.hpp) -----------------------------------
void* tsylv_rng_new(std::uint64_t seed) { return new RandomStream(seed); }
void tsylv_rng_free(void* r) { delete static_cast<RandomStream*>(r); }
double tsylv_rng_uniform(void* r) { return static_cast<RandomStream*>(r)->uniform(); }
double tsylv_rng_normal(void* r) { return static_cast<RandomStream*>(r)->normal(); }
void tsylv_rng_randn(void* r, double* out, size_t n) {
  auto* s = static_cast<RandomStream*>(r);
  for (size_t i = 0; i < n; ++i) out[i] = s->normal();
}

// BASELINE.json configuration generator: kind 1/2 Laplace (coeffs packed
// back to back, c unused), kind 5 gsylv.  Returns 0 or TSG_EDIM.
int tsylv_make_problem(int kind, int d, const int* dims, std::uint64_t seed, double* coeffs,
                       double* c, double* rhs) {
  if (d < 2) return TSG_EDIM;
  if (kind == 1 || kind == 2) {
    LaplaceProblem<double> p = baseline_laplace(kind, dv(d, dims), seed);
    for (int m = 0; m < d; ++m) {
      std::memcpy(coeffs, p.coeffs[m].data(), p.coeffs[m].size() * sizeof(double));
      coeffs += p.coeffs[m].size();
    }
    std::memcpy(rhs, p.rhs.data(), p.rhs.size() * sizeof(double));
    return TSG_OK;
  }
  if (kind == 5) {
    for (int m = 2; m < d; ++m)
      if (dims[m] != dims[1]) return TSG_EDIM;
    GSylvProblem<double> p = baseline_gsylv(dv(d, dims), seed);
    for (int m = 0; m < d; ++m) {
      std::memcpy(coeffs, p.coeffs[m].data(), p.coeffs[m].size() * sizeof(double));
      coeffs += p.coeffs[m].size();
    }
    std::memcpy(c, p.c.data(), p.c.size() * sizeof(double));
    std::memcpy(rhs, p.rhs.data(), p.rhs.size() * sizeof(double));
    return TSG_OK;
  }
  return TSG_EDIM;
}

// ---- T = Complex: interleaved complex buffers ------
int tsylv_zsolve_laplace(int d, const int* dims, const double* const* coeffs, const double* rhs,
                         int strategy, int arithmetic, int n_min, double* x, double* info,
                         char* err, int errlen) {
  return guarded(err, errlen, [&] {
    LaplaceProblem<Z> p;
    p.coeffs = zmats(d, dims, coeffs);
    p.rhs = zten(d, dims, rhs);
    SolveReport<Z> r = solve_laplace(p, cfg_of(strategy, arithmetic, n_min));
    zout(r.solution, x);
    zfill_info(r, info);
  });
}

int tsylv_zsolve_gsylv(int d, const int* dims, const double* const* coeffs, const double* c,
                       const double* rhs, int strategy, int arithmetic, int n_min, double* x,
                       double* info, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GSylvProblem<Z> p;
    p.coeffs = zmats(d, dims, coeffs);
    p.c = zmat(dims[0], dims[0], c);
    p.rhs = zten(d, dims, rhs);
    SolveReport<Z> r = solve_gsylv(p, cfg_of(strategy, arithmetic, n_min));
    zout(r.solution, x);
    zfill_info(r, info);
  });
}

int tsylv_zlaplace_recursive(int d, const int* dims, const double* const* t, const double* bt,
                             int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen,
                 [&] { zout(laplace_recursive(zmats(d, dims, t), zten(d, dims, bt), n_min), x); });
}

int tsylv_zlaplace_merged(int d, const int* dims, const double* const* t, const double* bt,
                          int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen,
                 [&] { zout(laplace_merged(zmats(d, dims, t), zten(d, dims, bt), n_min), x); });
}

int tsylv_zgsylv_recursive(int d, const int* dims, const double* const* t, const double* tc,
                           const double* bt, int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    zout(gsylv_recursive(zmats(d, dims, t), zmat(dims[0], dims[0], tc), zten(d, dims, bt), n_min),
         x);
  });
}

int tsylv_zgsylv_merged(int d, const int* dims, const double* const* t, const double* tc,
                        const double* bt, int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    zout(gsylv_merged(zmats(d, dims, t), zmat(dims[0], dims[0], tc), zten(d, dims, bt), n_min), x);
  });
}

int tsylv_zsolve_sylvester_tri(int r, int c, const double* a1, const double* a2, const double* b,
                               int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    zout(solve_sylvester_tri(zmat(r, r, a1), zmat(c, c, a2), zmat(r, c, b), n_min), x);
  });
}

int tsylv_zsolve_gsylv_tri(int r, int c, const double* a1, const double* cm, const double* a2,
                           const double* b, int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    zout(solve_gsylv_tri(zmat(r, r, a1), zmat(r, r, cm), zmat(c, c, a2), zmat(r, c, b), n_min), x);
  });
}

int tsylv_zoracle_solve_laplace(int d, const int* dims, const double* const* coeffs,
                                const double* rhs, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    LaplaceProblem<Z> p;
    p.coeffs = zmats(d, dims, coeffs);
    p.rhs = zten(d, dims, rhs);
    zout(oracle::solve(p), x);
  });
}

int tsylv_zoracle_solve_gsylv(int d, const int* dims, const double* const* coeffs, const double* c,
                              const double* rhs, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GSylvProblem<Z> p;
    p.coeffs = zmats(d, dims, coeffs);
    p.c = zmat(dims[0], dims[0], c);
    p.rhs = zten(d, dims, rhs);
    zout(oracle::solve(p), x);
  });
}

int tsylv_zmode_multiply(int d, const int* dims, const double* xin, int r, const double* a,
                         int mode, double* y, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    zout(mode_multiply(zten(d, dims, xin), zmat(r, dims[mode], a), mode), y);
  });
}

int tsylv_zschur(int n, const double* a, double* u, double* t, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    SchurFactorization<Z> f = schur(zmat(n, n, a));
    zout(f.u, u);
    zout(f.t, t);
  });
}

int tsylv_zqz(int n, const double* a, const double* c, double* q, double* z, double* s, double* t,
              char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GeneralizedSchurFactorization<Z> f = qz(zmat(n, n, a), zmat(n, n, c));
    zout(f.u, q);
    zout(f.z, z);
    zout(f.s, s);
    zout(f.t, t);
  });
}

double tsylv_zresidual_laplace(int d, const int* dims, const double* const* coeffs,
                               const double* rhs, const double* x) {
  LaplaceProblem<Z> p;
  p.coeffs = zmats(d, dims, coeffs);
  p.rhs = zten(d, dims, rhs);
  return oracle::residual(p, zten(d, dims, x));
}

double tsylv_zresidual_gsylv(int d, const int* dims, const double* const* coeffs, const double* c,
                             const double* rhs, const double* x) {
  GSylvProblem<Z> p;
  p.coeffs = zmats(d, dims, coeffs);
  p.c = zmat(dims[0], dims[0], c);
  p.rhs = zten(d, dims, rhs);
  return oracle::residual(p, zten(d, dims, x));
}

// Complex correctness-suite generators (random.hpp:64-223, T = Complex):
// which 0 random_laplace_problem, 1 random_reduced_laplace,
// 2 random_gsylv_problem, 3 random_reduced_gsylv.  Coefficients packed back
// to back, then C (gsylv), then rhs; interleaved.
void tsylv_zrandom_problem(void* r, int which, int d, const int* dims, double* coeffs, double* c,
                           double* rhs) {
  auto& rng = *static_cast<RandomStream*>(r);
  auto pack = [&](const auto& p) {
    for (const auto& a : p.coeffs) {
      zout(a, coeffs);
      coeffs += 2 * a.size();
    }
    zout(p.rhs, rhs);
  };
  if (which == 0) pack(random_laplace_problem<Z>(rng, dv(d, dims)));
  else if (which == 1) pack(random_reduced_laplace<Z>(rng, dv(d, dims)));
  else {
    GSylvProblem<Z> p = which == 2 ? random_gsylv_problem<Z>(rng, dv(d, dims))
                                   : random_reduced_gsylv<Z>(rng, dv(d, dims));
    zout(p.c, c);
    pack(p);
  }
}

}  // extern "C"
