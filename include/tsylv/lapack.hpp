// tsylv drop-in (B200 build) — shared host setup: real / complex Schur
// (dgees / zgees) and
// generalized Schur (dgges / zgges) of the small coefficient matrices, computed once
// with the same LAPACK the oracle links (BASELINE.json north_star: "the
// Schur/QZ factors ... are computed once as shared setup input").  Contract
// of the reference's schur/qz (kernels.hpp:78-156): A = U T U^T with T upper
// quasi-triangular; (A, C) = (Q S Z^T, Q T Z^T).  LAPACK failures raise
// factorization_error with info (kernels.hpp:67-75).
#pragma once
#include <algorithm>
#include <complex>
#include <string>
#include <vector>

#include "tsylv/errors.hpp"
#include "tsylv/matrix.hpp"

extern "C" {
void dgees_(const char* jobvs, const char* sort, void* select, const int* n, double* a,
            const int* lda, int* sdim, double* wr, double* wi, double* vs, const int* ldvs,
            double* work, const int* lwork, int* bwork, int* info);
void dgges_(const char* jobvsl, const char* jobvsr, const char* sort, void* selctg, const int* n,
            double* a, const int* lda, double* b, const int* ldb, int* sdim, double* alphar,
            double* alphai, double* beta, double* vsl, const int* ldvsl, double* vsr,
            const int* ldvsr, double* work, const int* lwork, int* bwork, int* info);
void zgees_(const char* jobvs, const char* sort, void* select, const int* n,
            std::complex<double>* a, const int* lda, int* sdim, std::complex<double>* w,
            std::complex<double>* vs, const int* ldvs, std::complex<double>* work,
            const int* lwork, double* rwork, int* bwork, int* info);
void zgges_(const char* jobvsl, const char* jobvsr, const char* sort, void* selctg, const int* n,
            std::complex<double>* a, const int* lda, std::complex<double>* b, const int* ldb,
            int* sdim, std::complex<double>* alpha, std::complex<double>* beta,
            std::complex<double>* vsl, const int* ldvsl, std::complex<double>* vsr,
            const int* ldvsr, std::complex<double>* work, const int* lwork, double* rwork,
            int* bwork, int* info);
}

namespace tsylv {

// T = double: real Schur (T quasi-triangular); T = Complex: complex Schur
// (T triangular, zgees / zgges), as the reference's templates.
template <typename T = double>
struct SchurFactorization {
  Matrix<T> u, t;
};
template <typename T = double>
struct GeneralizedSchurFactorization {
  Matrix<T> u, z, s, t;  // u = Q (left), z = Z (right)
};

namespace detail {
[[noreturn]] inline void lapack_error(const char* who, int info) {
  if (info < 0) throw std::invalid_argument(std::string(who) + ": illegal argument " + std::to_string(-info));
  throw factorization_error(std::string(who) + ": QR/QZ iteration failed to converge (info=" +
                                std::to_string(info) + ")",
                            info);
}
}  // namespace detail

inline SchurFactorization<double> schur(Matrix<double> a) {
  const int n = a.rows();
  if (n == 0 || n != a.cols()) throw dimension_error("schur: matrix must be square and non-empty");
  Matrix<double> vs(n, n);
  std::vector<double> wr(n), wi(n);
  int sdim = 0, info = 0, lw = -1;
  double q = 0;
  dgees_("V", "N", nullptr, &n, a.data(), &n, &sdim, wr.data(), wi.data(), vs.data(), &n, &q, &lw,
         nullptr, &info);
  lw = std::max(1, static_cast<int>(q));
  std::vector<double> work(lw);
  dgees_("V", "N", nullptr, &n, a.data(), &n, &sdim, wr.data(), wi.data(), vs.data(), &n,
         work.data(), &lw, nullptr, &info);
  if (info != 0) detail::lapack_error("dgees", info);
  return {std::move(vs), std::move(a)};
}

inline GeneralizedSchurFactorization<double> qz(Matrix<double> a, Matrix<double> c) {
  const int n = a.rows();
  if (n == 0 || n != a.cols()) throw dimension_error("qz: matrix must be square and non-empty");
  if (c.rows() != n || c.cols() != n) throw dimension_error("qz: pencil matrices must have equal shape");
  Matrix<double> l(n, n), r(n, n);
  std::vector<double> ar(n), ai(n), be(n);
  int sdim = 0, info = 0, lw = -1;
  double q = 0;
  dgges_("V", "V", "N", nullptr, &n, a.data(), &n, c.data(), &n, &sdim, ar.data(), ai.data(),
         be.data(), l.data(), &n, r.data(), &n, &q, &lw, nullptr, &info);
  lw = std::max(1, static_cast<int>(q));
  std::vector<double> work(lw);
  dgges_("V", "V", "N", nullptr, &n, a.data(), &n, c.data(), &n, &sdim, ar.data(), ai.data(),
         be.data(), l.data(), &n, r.data(), &n, work.data(), &lw, nullptr, &info);
  if (info != 0) detail::lapack_error("dgges", info);
  return {std::move(l), std::move(r), std::move(a), std::move(c)};
}

inline SchurFactorization<Complex> schur(Matrix<Complex> a) {
  const int n = a.rows();
  if (n == 0 || n != a.cols()) throw dimension_error("schur: matrix must be square and non-empty");
  Matrix<Complex> vs(n, n);
  std::vector<Complex> w(n);
  std::vector<double> rwork(n);
  int sdim = 0, info = 0, lw = -1;
  Complex q;
  zgees_("V", "N", nullptr, &n, a.data(), &n, &sdim, w.data(), vs.data(), &n, &q, &lw,
         rwork.data(), nullptr, &info);
  lw = std::max(1, static_cast<int>(q.real()));
  std::vector<Complex> work(lw);
  zgees_("V", "N", nullptr, &n, a.data(), &n, &sdim, w.data(), vs.data(), &n, work.data(), &lw,
         rwork.data(), nullptr, &info);
  if (info != 0) detail::lapack_error("zgees", info);
  return {std::move(vs), std::move(a)};
}

inline GeneralizedSchurFactorization<Complex> qz(Matrix<Complex> a, Matrix<Complex> c) {
  const int n = a.rows();
  if (n == 0 || n != a.cols()) throw dimension_error("qz: matrix must be square and non-empty");
  if (c.rows() != n || c.cols() != n) throw dimension_error("qz: pencil matrices must have equal shape");
  Matrix<Complex> l(n, n), r(n, n);
  std::vector<Complex> al(n), be(n);
  std::vector<double> rwork(8 * static_cast<size_t>(n));
  int sdim = 0, info = 0, lw = -1;
  Complex q;
  zgges_("V", "V", "N", nullptr, &n, a.data(), &n, c.data(), &n, &sdim, al.data(), be.data(),
         l.data(), &n, r.data(), &n, &q, &lw, rwork.data(), nullptr, &info);
  lw = std::max(1, static_cast<int>(q.real()));
  std::vector<Complex> work(lw);
  zgges_("V", "V", "N", nullptr, &n, a.data(), &n, c.data(), &n, &sdim, al.data(), be.data(),
         l.data(), &n, r.data(), &n, work.data(), &lw, rwork.data(), nullptr, &info);
  if (info != 0) detail::lapack_error("zgges", info);
  return {std::move(l), std::move(r), std::move(a), std::move(c)};
}

}  // namespace tsylv
