// tsylv drop-in (B200 build) — the host solvability screen run before the
// GPU solve so singular operators raise singular_error with the reference's
// witness semantics (solvability.hpp:31-116, laplace.hpp:28-43,
// gsylv.hpp:31-50): the smallest |operator eigenvalue| over every tuple, the
// first minimum in odometer order (mode 0 fastest).  The Laplace scan is
// split over host threads along the slowest mode; ties resolve to the lowest
// chunk, which keeps the sequential witness.
#pragma once
#include <algorithm>
#include <cmath>
#include <complex>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "tsylv/gpu.hpp"
#include "tsylv/matrix.hpp"
#include "tsylv/scalar.hpp"

namespace tsylv {

struct Solvability {
  bool solvable = true;
  double min_abs = 0;
  std::vector<int> witness;
  std::vector<std::complex<double>> witness_values;
};

using EigList = std::vector<std::complex<double>>;

// Eigenvalues of a quasi-triangular matrix in diagonal order.
inline EigList quasi_tri_eigenvalues(const Matrix<double>& t) {
  if (!is_upper_quasi_triangular(t))
    throw dimension_error("quasi_block_sizes: matrix is not upper quasi-triangular");
  using C = std::complex<double>;
  const int n = t.rows();
  EigList e;
  for (int j = 0; j < n;) {
    if (j + 1 < n && t(j + 1, j) != 0.0) {
      const C half_tr = 0.5 * (C(t(j, j)) + C(t(j + 1, j + 1)));
      const C det = C(t(j, j)) * C(t(j + 1, j + 1)) - C(t(j, j + 1)) * C(t(j + 1, j));
      const C r = std::sqrt(half_tr * half_tr - det);
      e.push_back(half_tr + r);
      e.push_back(half_tr - r);
      j += 2;
    } else {
      e.emplace_back(t(j, j));
      j += 1;
    }
  }
  return e;
}

// Complex (quasi-)triangular factors (complex Schur forms are triangular:
// the eigenvalues are the diagonal; 2x2 blocks keep the reference's exact
// block formula, kernels.hpp:309-330).
inline EigList quasi_tri_eigenvalues(const Matrix<std::complex<double>>& t) {
  if (!is_upper_quasi_triangular(t))
    throw dimension_error("quasi_block_sizes: matrix is not upper quasi-triangular");
  using C = std::complex<double>;
  const int n = t.rows();
  EigList e;
  for (int j = 0; j < n;) {
    if (j + 1 < n && t(j + 1, j) != C(0)) {
      const C tr = t(j, j) + t(j + 1, j + 1);
      const C det = t(j, j) * t(j + 1, j + 1) - t(j, j + 1) * t(j + 1, j);
      const C r = std::sqrt(tr * tr / 4.0 - det);
      e.push_back(tr / 2.0 + r);
      e.push_back(tr / 2.0 - r);
      j += 2;
    } else {
      e.push_back(t(j, j));
      j += 1;
    }
  }
  return e;
}

namespace detail {

inline Solvability min_kron_sum(const std::vector<EigList>& eigs) {
  using C = std::complex<double>;
  const int d = static_cast<int>(eigs.size());
  const int outer = static_cast<int>(eigs[d - 1].size());
  // Precompute the partial sums of modes 0..d-2 once (odometer order).
  std::vector<C> inner{C(0)};
  for (int m = 0; m + 1 < d; ++m) {
    std::vector<C> nx;
    nx.reserve(inner.size() * eigs[m].size());
    for (const C& l : eigs[m])
      for (const C& s : inner) nx.push_back(s + l);
    inner.swap(nx);
  }
  // Built newest-mode-outermost, i.e. index p enumerates modes 0..d-2 with
  // mode 0 fastest (the reference's odometer order).
  const std::vector<C>& ordered = inner;
  const int nt = std::max(1, std::min<int>(outer, static_cast<int>(std::thread::hardware_concurrency())));
  std::vector<double> best(nt, std::numeric_limits<double>::infinity());
  std::vector<size_t> best_in(nt, 0);
  std::vector<int> best_out(nt, 0);
  auto work = [&](int t) {
    for (int o = t; o < outer; o += nt) {
      const C l = eigs[d - 1][o];
      for (size_t p = 0; p < ordered.size(); ++p) {
        const double a = std::abs(ordered[p] + l);
        if (a < best[t] || (a == best[t] && (o < best_out[t] || (o == best_out[t] && p < best_in[t])))) {
          best[t] = a;
          best_in[t] = p;
          best_out[t] = o;
        }
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  int bt = 0;
  for (int t = 1; t < nt; ++t)
    if (best[t] < best[bt] || (best[t] == best[bt] && (best_out[t] < best_out[bt] ||
                                                      (best_out[t] == best_out[bt] && best_in[t] < best_in[bt]))))
      bt = t;
  Solvability s;
  s.min_abs = best[bt];
  size_t p = best_in[bt];
  for (int m = 0; m + 1 < d; ++m) {
    const size_t n = eigs[m].size();
    s.witness.push_back(static_cast<int>(p % n));
    p /= n;
  }
  s.witness.push_back(best_out[bt]);
  for (int m = 0; m < d; ++m) s.witness_values.push_back(eigs[m][s.witness[m]]);
  return s;
}

// Smallest eigenvalue magnitude of S_blk + z T_blk over the diagonal blocks
// of S and every product z of one tail eigenvalue per list.
inline Solvability min_pencil_product(const Matrix<double>& s_, const Matrix<double>& t_,
                                      const std::vector<EigList>& tails) {
  using C = std::complex<double>;
  const int n = s_.rows();
  std::vector<int> starts, sizes;
  for (int j = 0; j < n;) {
    const int sz = (j + 1 < n && s_(j + 1, j) != 0.0) ? 2 : 1;
    starts.push_back(j);
    sizes.push_back(sz);
    j += sz;
  }
  std::vector<C> prods{C(1)};
  for (const auto& l : tails) {
    std::vector<C> nx;
    for (const C& e : l)
      for (const C& p : prods) nx.push_back(p * e);
    prods.swap(nx);
  }
  Solvability out;
  out.min_abs = std::numeric_limits<double>::infinity();
  size_t best_p = 0;
  int best_b = 0;
  for (size_t p = 0; p < prods.size(); ++p) {
    const C z = prods[p];
    for (size_t b = 0; b < starts.size(); ++b) {
      const int i = starts[b];
      double mag;
      if (sizes[b] == 1) {
        mag = std::abs(C(s_(i, i)) + z * C(t_(i, i)));
      } else {
        const C m00 = C(s_(i, i)) + z * t_(i, i), m01 = C(s_(i, i + 1)) + z * t_(i, i + 1);
        const C m10 = C(s_(i + 1, i)), m11 = C(s_(i + 1, i + 1)) + z * t_(i + 1, i + 1);
        const C h = 0.5 * (m00 + m11);
        const C r = std::sqrt(h * h - (m00 * m11 - m01 * m10));
        mag = std::min(std::abs(h + r), std::abs(h - r));
      }
      if (mag < out.min_abs) {
        out.min_abs = mag;
        best_p = p;
        best_b = static_cast<int>(b);
      }
    }
  }
  out.witness.push_back(starts[best_b]);
  out.witness_values = {C(s_(starts[best_b], starts[best_b])), C(t_(starts[best_b], starts[best_b]))};
  size_t p = best_p;
  for (const auto& l : tails) {
    out.witness.push_back(static_cast<int>(p % l.size()));
    out.witness_values.push_back(l[p % l.size()]);
    p /= l.size();
  }
  return out;
}

// Complex pencil screen (solvability.hpp:65-116 with T = Complex): tuples
// in odometer order, blocks innermost, first strict minimum kept.
inline Solvability min_pencil_product(const Matrix<std::complex<double>>& a1,
                                      const Matrix<std::complex<double>>& c,
                                      const std::vector<EigList>& tails) {
  using C = std::complex<double>;
  const int n = a1.rows();
  std::vector<int> starts, sizes;
  for (int j = 0; j < n;) {
    const int sz = (j + 1 < n && a1(j + 1, j) != C(0)) ? 2 : 1;
    starts.push_back(j);
    sizes.push_back(sz);
    j += sz;
  }
  const int d = static_cast<int>(tails.size());
  Solvability out;
  out.min_abs = std::numeric_limits<double>::infinity();
  std::vector<int> idx(d, 0);
  for (;;) {
    C z = 1;
    for (int m = 0; m < d; ++m) z *= tails[m][idx[m]];
    for (size_t b = 0; b < starts.size(); ++b) {
      const int s0 = starts[b];
      double mag;
      if (sizes[b] == 1) {
        mag = std::abs(a1(s0, s0) + z * c(s0, s0));
      } else {
        const C m00 = a1(s0, s0) + z * c(s0, s0), m01 = a1(s0, s0 + 1) + z * c(s0, s0 + 1);
        const C m10 = a1(s0 + 1, s0), m11 = a1(s0 + 1, s0 + 1) + z * c(s0 + 1, s0 + 1);
        const C tr = m00 + m11;
        const C disc = std::sqrt(tr * tr / 4.0 - (m00 * m11 - m01 * m10));
        mag = std::min(std::abs(tr / 2.0 + disc), std::abs(tr / 2.0 - disc));
      }
      if (mag < out.min_abs) {
        out.min_abs = mag;
        out.witness.assign(1, s0);
        out.witness.insert(out.witness.end(), idx.begin(), idx.end());
        out.witness_values.assign({a1(s0, s0), c(s0, s0)});
        for (int m = 0; m < d; ++m) out.witness_values.push_back(tails[m][idx[m]]);
      }
    }
    int m = 0;
    while (m < d && ++idx[m] == static_cast<int>(tails[m].size())) {
      idx[m] = 0;
      ++m;
    }
    if (m == d) break;
  }
  return out;
}

inline std::string witness_message(const char* who, const Solvability& s) {
  std::string m = std::string(who) + ": operator numerically singular (|eigenvalue| = " +
                  std::to_string(s.min_abs) + " at slots (";
  for (size_t i = 0; i < s.witness.size(); ++i) m += (i ? "," : "") + std::to_string(s.witness[i]);
  return m + "))";
}

}  // namespace detail

inline Solvability check_solvable_laplace(const std::vector<Matrix<double>>& t, double tol = 0) {
  if (t.empty()) throw dimension_error("check_solvable_laplace: no coefficients");
  std::vector<EigList> e;
  double scale = 0;
  for (const auto& m : t) {
    e.push_back(quasi_tri_eigenvalues(m));
    scale += m.frobenius_norm();
  }
  if (tol <= 0) tol = unit_roundoff<double> * scale;
  Solvability s = detail::min_kron_sum(e);
  s.solvable = s.min_abs > tol;
  return s;
}

inline Solvability check_solvable_gsylv(const std::vector<Matrix<double>>& t,
                                        const Matrix<double>& c, double tol = 0) {
  if (t.size() < 2) throw dimension_error("check_solvable_gsylv: need at least two modes");
  if (c.rows() != t[0].rows() || c.cols() != t[0].cols())
    throw dimension_error("check_solvable_gsylv: C must match A_0");
  if (!is_upper_triangular(c)) throw dimension_error("check_solvable_gsylv: C must be upper triangular");
  double scale = t[0].frobenius_norm() + c.frobenius_norm();
  std::vector<EigList> tails;
  for (size_t m = 1; m < t.size(); ++m) {
    tails.push_back(quasi_tri_eigenvalues(t[m]));
    scale += t[m].frobenius_norm();
  }
  (void)quasi_tri_eigenvalues(t[0]);  // validates A_0
  if (tol <= 0) tol = unit_roundoff<double> * scale;
  Solvability s = detail::min_pencil_product(t[0], c, tails);
  s.solvable = s.min_abs > tol;
  return s;
}

// T = Complex (host scan; the GPU screens take real quasi-triangular factors).
inline Solvability check_solvable_laplace(const std::vector<Matrix<std::complex<double>>>& t,
                                          double tol = 0) {
  if (t.empty()) throw dimension_error("check_solvable_laplace: no coefficients");
  std::vector<EigList> e;
  double scale = 0;
  for (const auto& m : t) {
    e.push_back(quasi_tri_eigenvalues(m));
    scale += m.frobenius_norm();
  }
  if (tol <= 0) tol = unit_roundoff<double> * scale;
  Solvability s = detail::min_kron_sum(e);
  s.solvable = s.min_abs > tol;
  return s;
}

inline Solvability check_solvable_gsylv(const std::vector<Matrix<std::complex<double>>>& t,
                                        const Matrix<std::complex<double>>& c, double tol = 0) {
  if (t.size() < 2) throw dimension_error("check_solvable_gsylv: need at least two modes");
  if (c.rows() != t[0].rows() || c.cols() != t[0].cols())
    throw dimension_error("check_solvable_gsylv: C must match A_0");
  if (!is_upper_triangular(c)) throw dimension_error("check_solvable_gsylv: C must be upper triangular");
  double scale = t[0].frobenius_norm() + c.frobenius_norm();
  std::vector<EigList> tails;
  for (size_t m = 1; m < t.size(); ++m) {
    tails.push_back(quasi_tri_eigenvalues(t[m]));
    scale += t[m].frobenius_norm();
  }
  (void)quasi_tri_eigenvalues(t[0]);  // validates A_0
  if (tol <= 0) tol = unit_roundoff<double> * scale;
  Solvability s = detail::min_pencil_product(t[0], c, tails);
  s.solvable = s.min_abs > tol;
  return s;
}

// The same screens on the GPU (tsg_screen_laplace / tsg_screen_gsylv,
// csrc/screen.cu): identical tolerance, witness and witness values; the
// solve entry points use these (the reference runs the scan inside its timed
// recursion, laplace.hpp:271-274, gsylv.hpp:267-270).
inline Solvability screen_laplace_gpu(const std::vector<Matrix<double>>& t, double tol = 0) {
  if (t.empty()) throw dimension_error("check_solvable_laplace: no coefficients");
  std::vector<EigList> e;
  std::vector<int> dims;
  std::vector<const double*> tp;
  for (const auto& m : t) {
    e.push_back(quasi_tri_eigenvalues(m));  // validates the factor
    dims.push_back(m.rows());
    tp.push_back(m.data());
  }
  Solvability s;
  s.witness.assign(t.size(), 0);
  int ok = 0;
  gpu::check(tsg_screen_laplace(gpu::context(), static_cast<int>(t.size()), dims.data(), tp.data(), tol, &s.min_abs,
                                s.witness.data(), &ok),
             "check_solvable_laplace");
  s.solvable = ok != 0;
  for (size_t m = 0; m < t.size(); ++m) s.witness_values.push_back(e[m][s.witness[m]]);
  return s;
}

inline Solvability screen_gsylv_gpu(const std::vector<Matrix<double>>& t, const Matrix<double>& c, double tol = 0) {
  if (t.size() < 2) throw dimension_error("check_solvable_gsylv: need at least two modes");
  if (c.rows() != t[0].rows() || c.cols() != t[0].cols())
    throw dimension_error("check_solvable_gsylv: C must match A_0");
  if (!is_upper_triangular(c)) throw dimension_error("check_solvable_gsylv: C must be upper triangular");
  std::vector<EigList> tails;
  std::vector<int> dims{t[0].rows()};
  std::vector<const double*> tp;
  (void)quasi_tri_eigenvalues(t[0]);  // validates A_0
  for (size_t m = 1; m < t.size(); ++m) {
    tails.push_back(quasi_tri_eigenvalues(t[m]));
    dims.push_back(t[m].rows());
    tp.push_back(t[m].data());
  }
  Solvability s;
  s.witness.assign(t.size(), 0);
  int ok = 0;
  gpu::check(tsg_screen_gsylv(gpu::context(), static_cast<int>(t.size()), dims.data(), t[0].data(), c.data(),
                              tp.data(), tol, &s.min_abs, s.witness.data(), &ok),
             "check_solvable_gsylv");
  s.solvable = ok != 0;
  using C = std::complex<double>;
  s.witness_values = {C(t[0](s.witness[0], s.witness[0])), C(c(s.witness[0], s.witness[0]))};
  for (size_t m = 1; m < t.size(); ++m) s.witness_values.push_back(tails[m - 1][s.witness[m]]);
  return s;
}

}  // namespace tsylv
