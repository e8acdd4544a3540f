// Host setup of the eigen-decoupled Laplace solve (solve_fibre.cu).
//
// For a real Schur factor T (standardised 2x2 blocks, as dgees returns them)
// the real block-eigenbasis P (LAPACK dtrevc: real eigenvectors, and
// [Re v, Im v] for a complex pair) gives T P = P Lambda with Lambda block
// diagonal.  Folding P into the transforms (forward P^{-1} U^T, back U P)
// leaves Lambda in the reduced operator for every mode in S; only the free
// mode f keeps its triangular factor.  The rounding of the folded
// transforms grows with prod_{s in S} kappa_2(P_s), so S is admitted only
// when that product is at most kDecoupleKappa (measured: C3 at 2.2e7 gives
// residual 3.5e-14 and rel. error 2.1e-13 against the reference, C2 at
// 4e4 gives 3.8e-15 / 7.0e-14; tools/decouple_probe.py); otherwise the plan
// keeps the tile-DAG kernels.
#include "decouple.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>

extern "C" {
void dtrevc_(const char* side, const char* howmny, int* select, const int* n, const double* t,
             const int* ldt, double* vl, const int* ldvl, double* vr, const int* ldvr, const int* mm,
             int* m, double* work, int* info);
void dgetrf_(const int* m, const int* n, double* a, const int* lda, int* ipiv, int* info);
void dgetri_(const int* n, double* a, const int* lda, const int* ipiv, double* work,
             const int* lwork, int* info);
void dgemm_(const char* ta, const char* tb, const int* m, const int* n, const int* k,
            const double* alpha, const double* a, const int* lda, const double* b, const int* ldb,
            const double* beta, double* c, const int* ldc);
}

namespace tsg_impl {
namespace {

double at(const double* a, int n, int i, int j) { return a[i + static_cast<size_t>(j) * n]; }

// ||A||_2 by power iteration on A^T A (a lower estimate; 60 steps, +2 %).
double norm2(const std::vector<double>& a, int n) {
  std::vector<double> v(n, 1.0 / std::sqrt(static_cast<double>(n))), w(n), u(n);
  double s = 0;
  for (int it = 0; it < 60; ++it) {
    for (int i = 0; i < n; ++i) {
      double acc = 0;
      for (int j = 0; j < n; ++j) acc += at(a.data(), n, i, j) * v[j];
      w[i] = acc;
    }
    for (int j = 0; j < n; ++j) {
      double acc = 0;
      const double* cj = a.data() + static_cast<size_t>(j) * n;
      for (int i = 0; i < n; ++i) acc += cj[i] * w[i];
      u[j] = acc;
    }
    double nu = 0;
    for (double x : u) nu += x * x;
    nu = std::sqrt(nu);
    if (!(nu > 0) || !std::isfinite(nu)) return std::numeric_limits<double>::infinity();
    s = std::sqrt(nu);
    for (int j = 0; j < n; ++j) v[j] = u[j] / nu;
  }
  return std::isfinite(s) ? 1.02 * s : std::numeric_limits<double>::infinity();
}

}  // namespace

bool mode_eigen(const double* T, int n, ModeEigen& me) {
  me = ModeEigen{};
  me.n = n;
  // cells; every 2x2 block must carry a complex pair (LAPACK standard form)
  for (int i = 0; i < n;) {
    tsg::FibreCell c{};
    c.start = i;
    if (i + 1 < n && at(T, n, i + 1, i) != 0.0) {
      const double a = at(T, n, i, i), b = at(T, n, i, i + 1);
      const double cc = at(T, n, i + 1, i), d = at(T, n, i + 1, i + 1);
      const double disc = 0.25 * (a - d) * (a - d) + b * cc;
      if (!(disc < 0)) return false;
      c.size = 2;
      c.re = 0.5 * (a + d);
      c.im = std::sqrt(-disc);  // sign fixed below from P^{-1} T P
      i += 2;
    } else {
      c.size = 1;
      c.re = at(T, n, i, i);
      c.im = 0;
      i += 1;
    }
    me.cells.push_back(c);
  }
  // right eigenvectors of T in real format
  std::vector<double> vr(static_cast<size_t>(n) * n), work(3 * static_cast<size_t>(n));
  int mm = n, m = 0, info = 0, ld = n, one = 1;
  dtrevc_("R", "A", nullptr, &n, T, &ld, nullptr, &one, vr.data(), &ld, &mm, &m, work.data(), &info);
  if (info != 0 || m != n) return false;
  for (const auto& c : me.cells) {  // unit columns (a pair keeps its [Re, Im] ratio)
    double s = 0;
    for (int q = c.start; q < c.start + c.size; ++q)
      for (int i = 0; i < n; ++i) s += vr[i + static_cast<size_t>(q) * n] * vr[i + static_cast<size_t>(q) * n];
    s = std::sqrt(s / c.size);
    if (!(s > 0)) return false;
    for (int q = c.start; q < c.start + c.size; ++q)
      for (int i = 0; i < n; ++i) vr[i + static_cast<size_t>(q) * n] /= s;
  }
  std::vector<double> pinv = vr;
  std::vector<int> piv(n);
  dgetrf_(&n, &n, pinv.data(), &ld, piv.data(), &info);
  if (info != 0) return false;
  int lw = -1;
  double q = 0;
  dgetri_(&n, pinv.data(), &ld, piv.data(), &q, &lw, &info);
  lw = std::max(1, static_cast<int>(q));
  std::vector<double> wk(lw);
  dgetri_(&n, pinv.data(), &ld, piv.data(), wk.data(), &lw, &info);
  if (info != 0) return false;
  // Lambda = P^{-1} T P: sign of each pair's imaginary part, and a check
  // that the off-diagonal blocks vanish
  std::vector<double> tp(static_cast<size_t>(n) * n), lam(static_cast<size_t>(n) * n);
  const double o1 = 1.0, z0 = 0.0;
  dgemm_("N", "N", &n, &n, &n, &o1, T, &ld, vr.data(), &ld, &z0, tp.data(), &ld);
  dgemm_("N", "N", &n, &n, &n, &o1, pinv.data(), &ld, tp.data(), &ld, &z0, lam.data(), &ld);
  double tn = 0, off = 0;
  for (size_t i = 0; i < static_cast<size_t>(n) * n; ++i) tn += T[i] * T[i];
  tn = std::sqrt(tn);
  std::vector<int> cellof(n);
  for (int c = 0; c < static_cast<int>(me.cells.size()); ++c)
    for (int r = me.cells[c].start; r < me.cells[c].start + me.cells[c].size; ++r) cellof[r] = c;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      if (cellof[i] != cellof[j]) off = std::max(off, std::abs(at(lam.data(), n, i, j)));
  for (auto& c : me.cells)
    if (c.size == 2 && at(lam.data(), n, c.start, c.start + 1) < 0) c.im = -c.im;
  for (double v : pinv)
    if (!std::isfinite(v)) return false;
  me.kappa = norm2(vr, n) * norm2(pinv, n);
  if (!(me.kappa < 1e300)) return false;
  // the diagonalisation must hold to ~kappa ulps of ||T||
  if (!(off <= 1e-14 * me.kappa * tn * n) && !(off <= 1e-9 * tn)) return false;
  me.P = std::move(vr);
  me.Pinv = std::move(pinv);
  return std::isfinite(me.kappa);
}

std::vector<double> matmul(const double* a, const double* b, int n) {
  std::vector<double> c(static_cast<size_t>(n) * n);
  const double o1 = 1.0, z0 = 0.0;
  dgemm_("N", "N", &n, &n, &n, &o1, a, &n, b, &n, &z0, c.data(), &n);
  return c;
}

}  // namespace tsg_impl
