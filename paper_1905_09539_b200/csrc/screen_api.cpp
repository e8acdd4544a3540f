// C-ABI of the GPU solvability screen (screen.cu): tsg_screen_laplace /
// tsg_screen_gsylv mirror check_solvable_laplace / check_solvable_gsylv of
// the reference (solvability.hpp:31-116): eigenvalues of the quasi-triangular
// factors in diagonal order (2x2 blocks by the same complex formula),
// tolerance unit_roundoff * (sum of Frobenius norms) when tol <= 0, the
// witness of the first minimum in the reference's scan order.
#include <cmath>
#include <complex>
#include <limits>
#include <vector>

#include "plan_impl.h"
#include "screen.h"
#include "tsylv_gpu.h"

namespace {

using C = std::complex<double>;

double at(const double* t, int n, int i, int j) { return t[i + static_cast<size_t>(j) * n]; }

// quasi_tri_eigenvalues (reference solvability.hpp), interleaved (re, im)
std::vector<double> eigenvalues(const double* t, int n) {
  std::vector<double> e;
  for (int j = 0; j < n;) {
    if (j + 1 < n && at(t, n, j + 1, j) != 0.0) {
      const C half_tr = 0.5 * (C(at(t, n, j, j)) + C(at(t, n, j + 1, j + 1)));
      const C det = C(at(t, n, j, j)) * C(at(t, n, j + 1, j + 1)) - C(at(t, n, j, j + 1)) * C(at(t, n, j + 1, j));
      const C r = std::sqrt(half_tr * half_tr - det);
      for (const C& v : {half_tr + r, half_tr - r}) {
        e.push_back(v.real());
        e.push_back(v.imag());
      }
      j += 2;
    } else {
      e.push_back(at(t, n, j, j));
      e.push_back(0.0);
      j += 1;
    }
  }
  return e;
}

double fro(const double* a, size_t n) {
  double s = 0;
  for (size_t i = 0; i < n; ++i) s += a[i] * a[i];
  return std::sqrt(s);
}

int nsm_of(int device) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  return n > 0 ? n : 148;
}

}  // namespace

extern "C" {

int tsg_screen_laplace(tsg_ctx* ctx, int d, const int* dims, const double* const* T, double tol,
                       double* min_abs, int* witness, int* solvable) {
  if (!ctx || !dims || !T || !min_abs || !solvable) return TSG_EINVAL;
  if (d < 1 || d > TSG_MAX_ORDER) return tsg_impl::fail(ctx, TSG_EDIM, "screen: order out of range");
  TSG_CU(cudaSetDevice(ctx->device));
  std::vector<std::vector<double>> e(d);
  tsg::ScreenSpec sp;
  sp.nlists = d;
  double scale = 0;
  for (int m = 0; m < d; ++m) {
    if (dims[m] <= 0) return tsg_impl::fail(ctx, TSG_EDIM, "screen: dimensions must be positive");
    e[m] = eigenvalues(T[m], dims[m]);
    sp.n[m] = dims[m];
    sp.eig_re_im[m] = e[m].data();
    scale += fro(T[m], static_cast<size_t>(dims[m]) * dims[m]);
  }
  sp.nsm = nsm_of(ctx->device);
  if (tol <= 0) tol = 0.5 * std::numeric_limits<double>::epsilon() * scale;
  int64_t idx = 0;
  TSG_CU(tsg::screen_min(sp, ctx->stream, min_abs, &idx));
  *solvable = *min_abs > tol ? 1 : 0;
  if (witness)
    for (int m = 0; m < d; ++m) {
      witness[m] = static_cast<int>(idx % dims[m]);
      idx /= dims[m];
    }
  return TSG_OK;
}

int tsg_screen_gsylv(tsg_ctx* ctx, int d, const int* dims, const double* S, const double* Tc,
                     const double* const* Ttail, double tol, double* min_abs, int* witness, int* solvable) {
  if (!ctx || !dims || !S || !Tc || !min_abs || !solvable || (d > 1 && !Ttail)) return TSG_EINVAL;
  if (d < 2 || d > TSG_MAX_ORDER) return tsg_impl::fail(ctx, TSG_EDIM, "screen: need at least two modes");
  TSG_CU(cudaSetDevice(ctx->device));
  const int n0 = dims[0];
  std::vector<std::vector<double>> e(d - 1);
  tsg::ScreenSpec sp;
  sp.nlists = d - 1;
  double scale = fro(S, static_cast<size_t>(n0) * n0) + fro(Tc, static_cast<size_t>(n0) * n0);
  for (int m = 1; m < d; ++m) {
    e[m - 1] = eigenvalues(Ttail[m - 1], dims[m]);
    sp.n[m - 1] = dims[m];
    sp.eig_re_im[m - 1] = e[m - 1].data();
    scale += fro(Ttail[m - 1], static_cast<size_t>(dims[m]) * dims[m]);
  }
  std::vector<int> starts, sizes;
  for (int j = 0; j < n0;) {
    const int sz = (j + 1 < n0 && at(S, n0, j + 1, j) != 0.0) ? 2 : 1;
    starts.push_back(j);
    sizes.push_back(sz);
    j += sz;
  }
  sp.S = S;
  sp.Tc = Tc;
  sp.n0 = n0;
  sp.nblk = static_cast<int>(starts.size());
  sp.bstart = starts.data();
  sp.bsize = sizes.data();
  sp.nsm = nsm_of(ctx->device);
  if (tol <= 0) tol = 0.5 * std::numeric_limits<double>::epsilon() * scale;
  int64_t idx = 0;
  TSG_CU(tsg::screen_min(sp, ctx->stream, min_abs, &idx));
  *solvable = *min_abs > tol ? 1 : 0;
  if (witness) {
    witness[0] = starts[static_cast<size_t>(idx % sp.nblk)];
    idx /= sp.nblk;
    for (int m = 1; m < d; ++m) {
      witness[m] = static_cast<int>(idx % dims[m]);
      idx /= dims[m];
    }
  }
  return TSG_OK;
}

}  // extern "C"
