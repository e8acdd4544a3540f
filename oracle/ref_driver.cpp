// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// Thin extern "C" driver around the UNMODIFIED reference headers under
// /root/reference/proj/include (compiled in place by oracle/Makefile, output
// only to oracle/_ref/).  It exposes the reference's own entry points so the
// pytest suite, the golden-fixture generator and bench.py's CPU baseline leg
// can call the reference CPU solver through ctypes:
//   solve_laplace       laplace.hpp:324-344
//   solve_gsylv         gsylv.hpp:311-331
//   laplace_recursive   laplace.hpp:185-195
//   gsylv_recursive     gsylv.hpp:149-159
//   laplace_merged      laplace.hpp:202-244
//   gsylv_merged        gsylv.hpp:167-232
//   solve_sylvester_tri sylvester.hpp:194-215
//   solve_gsylv_tri     sylvester.hpp:219-241
//   mode_multiply       tensor.hpp:187-231
//   schur / qz          kernels.hpp:78-156
//   oracle::solve       oracle.hpp:205-221
//   oracle::residual    oracle.hpp:233-268
//   RandomStream        random.hpp:19-62 (+ generators :64-223)
//   BASELINE.json inputs (ref_baseline_problem): the configurations' formulas
//   drawn from the reference's own RandomStream / randn_matrix / randn_tensor,
//   so the reference arm of bench.py never loads the product library.
// Status codes follow the C-ABI convention of include/tsylv_gpu.h:
//   0 ok, 1 dimension_error, 2 singular_error, 3 factorization_error,
//   4 std::invalid_argument (config conflict), 5 anything else.
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "tsylv/gsylv.hpp"
#include "tsylv/laplace.hpp"
#include "tsylv/oracle.hpp"
#include "tsylv/random.hpp"
#ifdef REF_HAVE_JSON
#include "tsylv/bench.hpp"  // run_verify (bench.hpp:255-352); needs nlohmann/json
#endif

using namespace tsylv;

namespace {

void set_err(char* err, int errlen, const std::string& msg) {
  if (!err || errlen <= 0) return;
  std::strncpy(err, msg.c_str(), static_cast<std::size_t>(errlen - 1));
  err[errlen - 1] = 0;
}

template <typename F>
int guarded(char* err, int errlen, F&& fn) {
  try {
    fn();
    return 0;
  } catch (const dimension_error& e) {
    set_err(err, errlen, e.what());
    return 1;
  } catch (const singular_error& e) {
    set_err(err, errlen, e.what());
    return 2;
  } catch (const factorization_error& e) {
    set_err(err, errlen, e.what());
    return 3;
  } catch (const std::invalid_argument& e) {
    set_err(err, errlen, e.what());
    return 4;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return 5;
  }
}

std::vector<int> dims_of(int d, const int* dims) { return {dims, dims + d}; }

std::size_t numel(int d, const int* dims) {
  std::size_t n = 1;
  for (int i = 0; i < d; ++i) n *= static_cast<std::size_t>(dims[i]);
  return n;
}

Matrix<double> mat(int r, int c, const double* p) {
  return Matrix<double>(r, c, std::vector<double>(p, p + static_cast<std::size_t>(r) * c));
}

Tensor<double> ten(int d, const int* dims, const double* p) {
  return Tensor<double>(dims_of(d, dims), std::vector<double>(p, p + numel(d, dims)));
}

void copy_out(const Tensor<double>& t, double* out) {
  std::memcpy(out, t.data(), t.size() * sizeof(double));
}

SolverConfig make_cfg(int strategy, int arithmetic, int n_min) {
  SolverConfig cfg;
  cfg.n_min = n_min;
  cfg.strategy = strategy == 0 ? Strategy::recursion_only : Strategy::merge;
  cfg.arithmetic = arithmetic == 0 ? Arithmetic::complex_triangular
                                   : Arithmetic::real_quasitriangular;
  return cfg;
}

void fill_info(const SolveReport<double>& rep, double* info) {
  if (!info) return;
  info[0] = rep.residual;
  info[1] = rep.discarded_imag;
  info[2] = rep.timings.reduction_s;
  info[3] = rep.timings.recursion_s;
  info[4] = rep.timings.back_transform_s;
  info[5] = rep.n_min;
}

// ---- complex (T = Complex) helpers: buffers are interleaved (re, im)
// doubles, the layout of std::complex<double> arrays.
using C = std::complex<double>;
const C* cp(const double* p) { return reinterpret_cast<const C*>(p); }
Matrix<C> zmat(int r, int c, const double* p) {
  return Matrix<C>(r, c, std::vector<C>(cp(p), cp(p) + static_cast<std::size_t>(r) * c));
}
Tensor<C> zten(int d, const int* dims, const double* p) {
  return Tensor<C>(dims_of(d, dims), std::vector<C>(cp(p), cp(p) + numel(d, dims)));
}
void zcopy_out(const Tensor<C>& t, double* out) {
  std::memcpy(out, t.data(), t.size() * sizeof(C));
}
void zfill_info(const SolveReport<C>& rep, double* info) {
  if (!info) return;
  info[0] = rep.residual;
  info[1] = rep.discarded_imag;
  info[2] = rep.timings.reduction_s;
  info[3] = rep.timings.recursion_s;
  info[4] = rep.timings.back_transform_s;
  info[5] = rep.n_min;
}
std::vector<Matrix<C>> zcoeffs(int d, const int* dims, const double* const* t) {
  std::vector<Matrix<C>> v;
  for (int m = 0; m < d; ++m) v.push_back(zmat(dims[m], dims[m], t[m]));
  return v;
}
template <typename P>
void zpack(const P& p, double* coeffs, double* rhs) {
  for (const auto& a : p.coeffs) {
    std::memcpy(coeffs, a.data(), a.size() * sizeof(C));
    coeffs += 2 * a.size();
  }
  zcopy_out(p.rhs, rhs);
}

} // namespace

extern "C" {

// strategy: 0 recursion_only, 1 merge; arithmetic: 0 complex, 1 real.
int ref_solve_laplace(int d, const int* dims, const double* const* coeffs,
                      const double* rhs, int strategy, int arithmetic,
                      int n_min, double* x, double* info, char* err,
                      int errlen) {
  return guarded(err, errlen, [&] {
    LaplaceProblem<double> p;
    for (int m = 0; m < d; ++m) p.coeffs.push_back(mat(dims[m], dims[m], coeffs[m]));
    p.rhs = ten(d, dims, rhs);
    SolveReport<double> rep = solve_laplace(p, make_cfg(strategy, arithmetic, n_min));
    copy_out(rep.solution, x);
    fill_info(rep, info);
  });
}

int ref_solve_gsylv(int d, const int* dims, const double* const* coeffs,
                    const double* c, const double* rhs, int strategy,
                    int arithmetic, int n_min, double* x, double* info,
                    char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GSylvProblem<double> p;
    for (int m = 0; m < d; ++m) p.coeffs.push_back(mat(dims[m], dims[m], coeffs[m]));
    p.c = mat(dims[0], dims[0], c);
    p.rhs = ten(d, dims, rhs);
    SolveReport<double> rep = solve_gsylv(p, make_cfg(strategy, arithmetic, n_min));
    copy_out(rep.solution, x);
    fill_info(rep, info);
  });
}

int ref_laplace_recursive(int d, const int* dims, const double* const* t,
                          const double* bt, int n_min, double* x, char* err,
                          int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Matrix<double>> coeffs;
    for (int m = 0; m < d; ++m) coeffs.push_back(mat(dims[m], dims[m], t[m]));
    copy_out(laplace_recursive(coeffs, ten(d, dims, bt), n_min), x);
  });
}

int ref_gsylv_recursive(int d, const int* dims, const double* const* t,
                        const double* tc, const double* bt, int n_min,
                        double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Matrix<double>> coeffs;
    for (int m = 0; m < d; ++m) coeffs.push_back(mat(dims[m], dims[m], t[m]));
    copy_out(gsylv_recursive(coeffs, mat(dims[0], dims[0], tc), ten(d, dims, bt), n_min), x);
  });
}

int ref_laplace_merged(int d, const int* dims, const double* const* t,
                       const double* bt, int n_min, double* x, char* err,
                       int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Matrix<double>> coeffs;
    for (int m = 0; m < d; ++m) coeffs.push_back(mat(dims[m], dims[m], t[m]));
    copy_out(laplace_merged(std::move(coeffs), ten(d, dims, bt), n_min), x);
  });
}

int ref_gsylv_merged(int d, const int* dims, const double* const* t,
                     const double* tc, const double* bt, int n_min, double* x,
                     char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Matrix<double>> coeffs;
    for (int m = 0; m < d; ++m) coeffs.push_back(mat(dims[m], dims[m], t[m]));
    copy_out(gsylv_merged(std::move(coeffs), mat(dims[0], dims[0], tc), ten(d, dims, bt), n_min),
             x);
  });
}

// A1 X + X A2^H = B (a1: r x r, a2: c x c, b: r x c).
int ref_solve_sylvester_tri(int r, int c, const double* a1, const double* a2,
                            const double* b, int n_min, double* x, char* err,
                            int errlen) {
  return guarded(err, errlen, [&] {
    Matrix<double> out = solve_sylvester_tri(mat(r, r, a1), mat(c, c, a2), mat(r, c, b), n_min);
    std::memcpy(x, out.data(), out.size() * sizeof(double));
  });
}

// A1 X + C X A2^H = B.
int ref_solve_gsylv_tri(int r, int c, const double* a1, const double* cm,
                        const double* a2, const double* b, int n_min, double* x,
                        char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Matrix<double> out = solve_gsylv_tri(mat(r, r, a1), mat(r, r, cm), mat(c, c, a2),
                                         mat(r, c, b), n_min);
    std::memcpy(x, out.data(), out.size() * sizeof(double));
  });
}

int ref_mode_multiply(int d, const int* dims, const double* xin, int r,
                      const double* a, int mode, double* y, char* err,
                      int errlen) {
  return guarded(err, errlen, [&] {
    copy_out(mode_multiply(ten(d, dims, xin), mat(r, dims[mode], a), mode), y);
  });
}

int ref_schur(int n, const double* a, double* u, double* t, char* err,
              int errlen) {
  return guarded(err, errlen, [&] {
    SchurFactorization<double> f = schur(mat(n, n, a));
    std::memcpy(u, f.u.data(), f.u.size() * sizeof(double));
    std::memcpy(t, f.t.data(), f.t.size() * sizeof(double));
  });
}

int ref_qz(int n, const double* a, const double* c, double* q, double* z,
           double* s, double* t, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GeneralizedSchurFactorization<double> f = qz(mat(n, n, a), mat(n, n, c));
    std::memcpy(q, f.u.data(), f.u.size() * sizeof(double));
    std::memcpy(z, f.z.data(), f.z.size() * sizeof(double));
    std::memcpy(s, f.s.data(), f.s.size() * sizeof(double));
    std::memcpy(t, f.t.data(), f.t.size() * sizeof(double));
  });
}

int ref_dense_solve_laplace(int d, const int* dims, const double* const* coeffs,
                            const double* rhs, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    LaplaceProblem<double> p;
    for (int m = 0; m < d; ++m) p.coeffs.push_back(mat(dims[m], dims[m], coeffs[m]));
    p.rhs = ten(d, dims, rhs);
    copy_out(oracle::solve(p), x);
  });
}

int ref_dense_solve_gsylv(int d, const int* dims, const double* const* coeffs,
                          const double* c, const double* rhs, double* x,
                          char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GSylvProblem<double> p;
    for (int m = 0; m < d; ++m) p.coeffs.push_back(mat(dims[m], dims[m], coeffs[m]));
    p.c = mat(dims[0], dims[0], c);
    p.rhs = ten(d, dims, rhs);
    copy_out(oracle::solve(p), x);
  });
}

double ref_residual_laplace(int d, const int* dims, const double* const* coeffs,
                            const double* rhs, const double* x) {
  LaplaceProblem<double> p;
  for (int m = 0; m < d; ++m) p.coeffs.push_back(mat(dims[m], dims[m], coeffs[m]));
  p.rhs = ten(d, dims, rhs);
  return oracle::residual(p, ten(d, dims, x));
}

double ref_residual_gsylv(int d, const int* dims, const double* const* coeffs,
                          const double* c, const double* rhs, const double* x) {
  GSylvProblem<double> p;
  for (int m = 0; m < d; ++m) p.coeffs.push_back(mat(dims[m], dims[m], coeffs[m]));
  p.c = mat(dims[0], dims[0], c);
  p.rhs = ten(d, dims, rhs);
  return oracle::residual(p, ten(d, dims, x));
}

// Solvability screen (laplace.hpp:28-43 / gsylv.hpp:31-50) on reduced
// coefficients; returns min_abs and writes the witness slots.
int ref_check_solvable_laplace(int d, const int* dims, const double* const* t,
                               double tol, double* min_abs, int* witness,
                               int* solvable, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Matrix<double>> coeffs;
    for (int m = 0; m < d; ++m) coeffs.push_back(mat(dims[m], dims[m], t[m]));
    Solvability s = check_solvable_laplace(coeffs, tol);
    *min_abs = s.min_abs;
    *solvable = s.solvable ? 1 : 0;
    for (std::size_t i = 0; i < s.witness.size(); ++i) witness[i] = s.witness[i];
  });
}

int ref_check_solvable_gsylv(int d, const int* dims, const double* const* t, const double* c,
                             double tol, double* min_abs, int* witness, int* solvable, char* err,
                             int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Matrix<double>> coeffs;
    for (int m = 0; m < d; ++m) coeffs.push_back(mat(dims[m], dims[m], t[m]));
    Solvability s = check_solvable_gsylv(coeffs, mat(dims[0], dims[0], c), tol);
    *min_abs = s.min_abs;
    *solvable = s.solvable ? 1 : 0;
    for (std::size_t i = 0; i < s.witness.size(); ++i) witness[i] = s.witness[i];
  });
}

// ---- RandomStream (random.hpp:19-77) ------------------------------------
void* ref_rng_new(std::uint64_t seed) { return new RandomStream(seed); }
void ref_rng_free(void* r) { delete static_cast<RandomStream*>(r); }
double ref_rng_uniform(void* r) { return static_cast<RandomStream*>(r)->uniform(); }
double ref_rng_normal(void* r) { return static_cast<RandomStream*>(r)->normal(); }
void ref_rng_randn(void* r, double* out, std::size_t n) {
  auto* s = static_cast<RandomStream*>(r);
  for (std::size_t i = 0; i < n; ++i) out[i] = s->normal();
}

// Correctness-suite generators (random.hpp:79-223).  Outputs: coefficient
// blocks packed back to back (column-major), then C (gsylv), then rhs.
void ref_random_reduced_laplace(void* r, int d, const int* dims, double* coeffs,
                                double* rhs) {
  auto p = random_reduced_laplace<double>(*static_cast<RandomStream*>(r), dims_of(d, dims));
  for (int m = 0; m < d; ++m) {
    std::memcpy(coeffs, p.coeffs[m].data(), p.coeffs[m].size() * sizeof(double));
    coeffs += p.coeffs[m].size();
  }
  copy_out(p.rhs, rhs);
}

void ref_random_laplace_problem(void* r, int d, const int* dims, double* coeffs,
                                double* rhs) {
  auto p = random_laplace_problem<double>(*static_cast<RandomStream*>(r), dims_of(d, dims));
  for (int m = 0; m < d; ++m) {
    std::memcpy(coeffs, p.coeffs[m].data(), p.coeffs[m].size() * sizeof(double));
    coeffs += p.coeffs[m].size();
  }
  copy_out(p.rhs, rhs);
}

void ref_random_reduced_gsylv(void* r, int d, const int* dims, double* coeffs,
                              double* c, double* rhs) {
  auto p = random_reduced_gsylv<double>(*static_cast<RandomStream*>(r), dims_of(d, dims));
  for (int m = 0; m < d; ++m) {
    std::memcpy(coeffs, p.coeffs[m].data(), p.coeffs[m].size() * sizeof(double));
    coeffs += p.coeffs[m].size();
  }
  std::memcpy(c, p.c.data(), p.c.size() * sizeof(double));
  copy_out(p.rhs, rhs);
}

void ref_random_gsylv_problem(void* r, int d, const int* dims, double* coeffs,
                              double* c, double* rhs) {
  auto p = random_gsylv_problem<double>(*static_cast<RandomStream*>(r), dims_of(d, dims));
  for (int m = 0; m < d; ++m) {
    std::memcpy(coeffs, p.coeffs[m].data(), p.coeffs[m].size() * sizeof(double));
    coeffs += p.coeffs[m].size();
  }
  std::memcpy(c, p.c.data(), p.c.size() * sizeof(double));
  copy_out(p.rhs, rhs);
}

void ref_randn_quasi_triangular(void* r, int n, double diag_shift,
                                double pair_prob, double* out) {
  Matrix<double> m = randn_quasi_triangular(*static_cast<RandomStream*>(r), n,
                                            diag_shift, pair_prob);
  std::memcpy(out, m.data(), m.size() * sizeof(double));
}

// BASELINE.json configurations (kind 1: convection-diffusion Laplace, C1;
// kind 2: A = G/sqrt(n) + 3I Laplace, C2-C4; kind 5: gsylv A = G_A/sqrt(n0)
// + 4I, B = G_B/sqrt(n0), C = G_C/(2 sqrt(nc)), posed as coeffs {A, C^T, ..},
// c = B, C5).  Draw order: coefficients in mode order, then the rhs.  Output
// layout as the generators above.  Returns 1 on a bad kind.
int ref_baseline_problem(int kind, int d, const int* dims, std::uint64_t seed,
                         double* coeffs, double* c, double* rhs) {
  RandomStream r(seed);
  std::vector<Matrix<double>> co;
  Matrix<double> cc;
  if (kind == 1 || kind == 2) {
    for (int m = 0; m < d; ++m) {
      const int n = dims[m];
      Matrix<double> a(n, n);
      if (kind == 1) {
        const double cm = 0.5 + 1.5 * r.uniform();
        const double h2 = static_cast<double>(n + 1) * (n + 1), h1 = cm * (n + 1) / 2.0;
        for (int i = 0; i < n; ++i) {
          a(i, i) = 2.0 * h2;
          if (i + 1 < n) {
            a(i, i + 1) = -h2 + h1;
            a(i + 1, i) = -h2 - h1;
          }
        }
      } else {
        a = randn_matrix<double>(r, n, n);
        const double s = std::sqrt(static_cast<double>(n));
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i) a(i, j) /= s;
        for (int i = 0; i < n; ++i) a(i, i) += 3.0;
      }
      co.push_back(std::move(a));
    }
  } else if (kind == 5) {
    const int n0 = dims[0], nc = dims[1];
    Matrix<double> a = randn_matrix<double>(r, n0, n0);
    Matrix<double> b = randn_matrix<double>(r, n0, n0);
    Matrix<double> g = randn_matrix<double>(r, nc, nc);
    const double s0 = std::sqrt(static_cast<double>(n0));
    const double sc = 2.0 * std::sqrt(static_cast<double>(nc));
    for (int j = 0; j < n0; ++j)
      for (int i = 0; i < n0; ++i) {
        a(i, j) /= s0;
        b(i, j) /= s0;
      }
    for (int i = 0; i < n0; ++i) a(i, i) += 4.0;
    for (int j = 0; j < nc; ++j)
      for (int i = 0; i < nc; ++i) g(i, j) /= sc;
    co.push_back(std::move(a));
    const Matrix<double> gt = transposed(g);
    for (int m = 1; m < d; ++m) co.push_back(gt);
    cc = std::move(b);
  } else {
    return 1;
  }
  Tensor<double> t = randn_tensor<double>(r, dims_of(d, dims));
  for (int m = 0; m < d; ++m) {
    std::memcpy(coeffs, co[m].data(), co[m].size() * sizeof(double));
    coeffs += co[m].size();
  }
  if (kind == 5 && c) std::memcpy(c, cc.data(), cc.size() * sizeof(double));
  copy_out(t, rhs);
  return 0;
}

// ---- complex scalars (T = Complex): the same entry points on
// LaplaceProblem<Complex> / GSylvProblem<Complex> (laplace.hpp:324-344,
// gsylv.hpp:311-331 with is_complex_v<T>), interleaved buffers.
int ref_zsolve_laplace(int d, const int* dims, const double* const* coeffs, const double* rhs,
                       int strategy, int arithmetic, int n_min, double* x, double* info,
                       char* err, int errlen) {
  return guarded(err, errlen, [&] {
    LaplaceProblem<C> p;
    p.coeffs = zcoeffs(d, dims, coeffs);
    p.rhs = zten(d, dims, rhs);
    SolveReport<C> rep = solve_laplace(p, make_cfg(strategy, arithmetic, n_min));
    zcopy_out(rep.solution, x);
    zfill_info(rep, info);
  });
}

int ref_zsolve_gsylv(int d, const int* dims, const double* const* coeffs, const double* c,
                     const double* rhs, int strategy, int arithmetic, int n_min, double* x,
                     double* info, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GSylvProblem<C> p;
    p.coeffs = zcoeffs(d, dims, coeffs);
    p.c = zmat(dims[0], dims[0], c);
    p.rhs = zten(d, dims, rhs);
    SolveReport<C> rep = solve_gsylv(p, make_cfg(strategy, arithmetic, n_min));
    zcopy_out(rep.solution, x);
    zfill_info(rep, info);
  });
}

int ref_zlaplace_recursive(int d, const int* dims, const double* const* t, const double* bt,
                           int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    zcopy_out(laplace_recursive(zcoeffs(d, dims, t), zten(d, dims, bt), n_min), x);
  });
}

int ref_zlaplace_merged(int d, const int* dims, const double* const* t, const double* bt,
                        int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    zcopy_out(laplace_merged(zcoeffs(d, dims, t), zten(d, dims, bt), n_min), x);
  });
}

int ref_zgsylv_recursive(int d, const int* dims, const double* const* t, const double* tc,
                         const double* bt, int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    zcopy_out(gsylv_recursive(zcoeffs(d, dims, t), zmat(dims[0], dims[0], tc), zten(d, dims, bt),
                              n_min),
              x);
  });
}

int ref_zgsylv_merged(int d, const int* dims, const double* const* t, const double* tc,
                      const double* bt, int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    zcopy_out(gsylv_merged(zcoeffs(d, dims, t), zmat(dims[0], dims[0], tc), zten(d, dims, bt),
                           n_min),
              x);
  });
}

int ref_zsolve_sylvester_tri(int r, int c, const double* a1, const double* a2, const double* b,
                             int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Matrix<C> out = solve_sylvester_tri(zmat(r, r, a1), zmat(c, c, a2), zmat(r, c, b), n_min);
    std::memcpy(x, out.data(), out.size() * sizeof(C));
  });
}

int ref_zsolve_gsylv_tri(int r, int c, const double* a1, const double* cm, const double* a2,
                         const double* b, int n_min, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Matrix<C> out = solve_gsylv_tri(zmat(r, r, a1), zmat(r, r, cm), zmat(c, c, a2),
                                    zmat(r, c, b), n_min);
    std::memcpy(x, out.data(), out.size() * sizeof(C));
  });
}

int ref_zmode_multiply(int d, const int* dims, const double* xin, int r, const double* a,
                       int mode, double* y, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    zcopy_out(mode_multiply(zten(d, dims, xin), zmat(r, dims[mode], a), mode), y);
  });
}

int ref_zschur(int n, const double* a, double* u, double* t, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    SchurFactorization<C> f = schur(zmat(n, n, a));
    std::memcpy(u, f.u.data(), f.u.size() * sizeof(C));
    std::memcpy(t, f.t.data(), f.t.size() * sizeof(C));
  });
}

int ref_zqz(int n, const double* a, const double* c, double* q, double* z, double* s, double* t,
            char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GeneralizedSchurFactorization<C> f = qz(zmat(n, n, a), zmat(n, n, c));
    std::memcpy(q, f.u.data(), f.u.size() * sizeof(C));
    std::memcpy(z, f.z.data(), f.z.size() * sizeof(C));
    std::memcpy(s, f.s.data(), f.s.size() * sizeof(C));
    std::memcpy(t, f.t.data(), f.t.size() * sizeof(C));
  });
}

int ref_zdense_solve_laplace(int d, const int* dims, const double* const* coeffs,
                             const double* rhs, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    LaplaceProblem<C> p;
    p.coeffs = zcoeffs(d, dims, coeffs);
    p.rhs = zten(d, dims, rhs);
    zcopy_out(oracle::solve(p), x);
  });
}

int ref_zdense_solve_gsylv(int d, const int* dims, const double* const* coeffs, const double* c,
                           const double* rhs, double* x, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GSylvProblem<C> p;
    p.coeffs = zcoeffs(d, dims, coeffs);
    p.c = zmat(dims[0], dims[0], c);
    p.rhs = zten(d, dims, rhs);
    zcopy_out(oracle::solve(p), x);
  });
}

double ref_zresidual_laplace(int d, const int* dims, const double* const* coeffs,
                             const double* rhs, const double* x) {
  LaplaceProblem<C> p;
  p.coeffs = zcoeffs(d, dims, coeffs);
  p.rhs = zten(d, dims, rhs);
  return oracle::residual(p, zten(d, dims, x));
}

double ref_zresidual_gsylv(int d, const int* dims, const double* const* coeffs, const double* c,
                           const double* rhs, const double* x) {
  GSylvProblem<C> p;
  p.coeffs = zcoeffs(d, dims, coeffs);
  p.c = zmat(dims[0], dims[0], c);
  p.rhs = zten(d, dims, rhs);
  return oracle::residual(p, zten(d, dims, x));
}

int ref_zcheck_solvable_laplace(int d, const int* dims, const double* const* t, double tol,
                                double* min_abs, int* witness, int* solvable, char* err,
                                int errlen) {
  return guarded(err, errlen, [&] {
    Solvability s = check_solvable_laplace(zcoeffs(d, dims, t), tol);
    *min_abs = s.min_abs;
    *solvable = s.solvable ? 1 : 0;
    for (std::size_t i = 0; i < s.witness.size(); ++i) witness[i] = s.witness[i];
  });
}

int ref_zcheck_solvable_gsylv(int d, const int* dims, const double* const* t, const double* c,
                              double tol, double* min_abs, int* witness, int* solvable, char* err,
                              int errlen) {
  return guarded(err, errlen, [&] {
    Solvability s = check_solvable_gsylv(zcoeffs(d, dims, t), zmat(dims[0], dims[0], c), tol);
    *min_abs = s.min_abs;
    *solvable = s.solvable ? 1 : 0;
    for (std::size_t i = 0; i < s.witness.size(); ++i) witness[i] = s.witness[i];
  });
}

// Complex generators (random.hpp:64-223 with T = Complex); layouts as the
// real ones, interleaved.
void ref_zrandn(void* r, double* out, std::size_t n) {
  auto* s = static_cast<RandomStream*>(r);
  for (std::size_t i = 0; i < n; ++i) {
    const C v = s->draw<C>();
    out[2 * i] = v.real();
    out[2 * i + 1] = v.imag();
  }
}
void ref_zrandom_reduced_laplace(void* r, int d, const int* dims, double* coeffs, double* rhs) {
  zpack(random_reduced_laplace<C>(*static_cast<RandomStream*>(r), dims_of(d, dims)), coeffs, rhs);
}
void ref_zrandom_laplace_problem(void* r, int d, const int* dims, double* coeffs, double* rhs) {
  zpack(random_laplace_problem<C>(*static_cast<RandomStream*>(r), dims_of(d, dims)), coeffs, rhs);
}
void ref_zrandom_reduced_gsylv(void* r, int d, const int* dims, double* coeffs, double* c,
                               double* rhs) {
  auto p = random_reduced_gsylv<C>(*static_cast<RandomStream*>(r), dims_of(d, dims));
  std::memcpy(c, p.c.data(), p.c.size() * sizeof(C));
  zpack(p, coeffs, rhs);
}
void ref_zrandom_gsylv_problem(void* r, int d, const int* dims, double* coeffs, double* c,
                               double* rhs) {
  auto p = random_gsylv_problem<C>(*static_cast<RandomStream*>(r), dims_of(d, dims));
  std::memcpy(c, p.c.data(), p.c.size() * sizeof(C));
  zpack(p, coeffs, rhs);
}

#ifdef REF_HAVE_JSON
// run_verify (bench.hpp:255-352): the seeded complex reduced-form suite;
// out: pass, instances, worst_rel, worst_residual.
int ref_run_verify(std::uint64_t seed, int per_family, const char* out_dir, double tol,
                   double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    VerifyReport v = run_verify(seed, per_family, out_dir ? out_dir : "", tol);
    out[0] = v.pass ? 1 : 0;
    out[1] = v.instances;
    out[2] = v.worst_rel;
    out[3] = v.worst_residual;
  });
}
#endif

} // extern "C"
