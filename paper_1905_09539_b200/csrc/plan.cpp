// C-ABI implementation (include/tsylv_gpu.h): contexts, plans, transforms.
//
// A plan is the device-resident form of one reduced problem: coefficient
// factors uploaded once, tile boundaries snapped off 2x2 Schur blocks
// (split_index rule, reference sylvester.hpp:43-49), per-block closed-form
// eigen data for the base cells, and the topological tile order of the
// dataflow solve.  tsg_plan_execute() then runs, on one stream:
//   forward transforms  B~ = B x_0 U_0^T x_1 U_1^T ...  (laplace.hpp:282;
//                       gsylv.hpp:278-280 with Q^T on mode 0)
//   reduced solve       (laplace.hpp:284-294 / gsylv.hpp:282-292)
//   back transforms     X = X~ x_0 U_0 ...              (laplace.hpp:297;
//                       gsylv.hpp:296-297 with Z on mode 0)
// captured once into a CUDA graph per (B, X) pointer pair.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/tsylv_gpu.h"
#include "gemm.h"
#include "solve.h"
#include "util.h"

#include "decouple.h"
#include "plan_impl.h"

namespace tsg_impl {

thread_local bool g_force_lap3 = false;

int fail(tsg_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

cudaError_t upload_mat(DevBuf& b, const double* h, size_t n) {
  cudaError_t e = b.ensure(n);
  if (e != cudaSuccess) return e;
  return cudaMemcpy(b.p, h, n * sizeof(double), cudaMemcpyHostToDevice);
}

std::vector<double> transpose(const double* a, int n) {
  std::vector<double> t(static_cast<size_t>(n) * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) t[j + static_cast<size_t>(i) * n] = a[i + static_cast<size_t>(j) * n];
  return t;
}

}  // namespace tsg_impl

namespace {

constexpr int kNoStatus = 0x7f7f7f7f;  // memset(0x7f) pattern: no singular cell

using tsg_impl::fail;
using tsg_impl::transpose;
using tsg_impl::upload_mat;

double at(const double* a, int n, int i, int j) { return a[i + static_cast<size_t>(j) * n]; }

// Exact structural predicates (matrix.hpp:152-172: no tolerance).
bool quasi_upper(const double* a, int n) {
  for (int j = 0; j < n; ++j)
    for (int i = j + 2; i < n; ++i)
      if (at(a, n, i, j) != 0.0) return false;
  for (int j = 0; j + 2 < n; ++j)
    if (at(a, n, j + 1, j) != 0.0 && at(a, n, j + 2, j + 1) != 0.0) return false;
  return true;
}
bool upper(const double* a, int n) {
  for (int j = 0; j < n; ++j)
    for (int i = j + 1; i < n; ++i)
      if (at(a, n, i, j) != 0.0) return false;
  return true;
}

double fro(const double* a, size_t n) {
  double s = 0;
  for (size_t i = 0; i < n; ++i) s += a[i] * a[i];
  return std::sqrt(s);
}

// Per-row block codes: 0 = 1x1, 1 = first row of a 2x2 block, 2 = second row.
std::vector<int8_t> block_codes(const double* t, int n) {
  std::vector<int8_t> c(n, 0);
  for (int i = 0; i < n;) {
    if (i + 1 < n && at(t, n, i + 1, i) != 0.0) {
      c[i] = 1;
      c[i + 1] = 2;
      i += 2;
    } else {
      i += 1;
    }
  }
  return c;
}

// Real normal form of every 2x2 diagonal block (kEigStride doubles at the
// block's first row; layout documented in solve.cu): a complex pair is
// W (alpha I + beta J) W^{-1} with W = [Re v, Im v] for the eigenvector v of
// alpha + i beta; a real pair is W diag(l0, l1) W^{-1}.  1x1 rows store t_ii.
// Returns false for a defective 2x2 block (equal real eigenvalues).
bool normal_form(const double* t, int n, const std::vector<int8_t>& code, std::vector<double>& e,
                 std::vector<double>& pdv, double* max_cond) {
  e.assign(static_cast<size_t>(n) * tsg::kEigStride, 0.0);
  pdv.assign(static_cast<size_t>(n) * tsg::kPStride, 0.0);
  for (int i = 0; i < n; ++i) {
    double* w = e.data() + static_cast<size_t>(i) * tsg::kEigStride;
    double* pr = pdv.data() + static_cast<size_t>(i) * tsg::kPStride;
    if (code[i] == 0) {
      w[0] = w[1] = at(t, n, i, i);
      w[4] = w[7] = w[8] = w[11] = 1.0;
      pr[0] = at(t, n, i, i);
      pr[4] = pr[10] = pr[12] = pr[18] = 1.0;  // P = Pinv = I
      continue;
    }
    if (code[i] != 1) continue;
    const double a = at(t, n, i, i), b = at(t, n, i, i + 1);
    const double c = at(t, n, i + 1, i), dd = at(t, n, i + 1, i + 1);
    const double h = 0.5 * (a + dd), disc = 0.25 * (a - dd) * (a - dd) + b * c;
    double W[4];  // row-major
    if (disc < 0) {
      const double beta = std::sqrt(-disc);
      // eigenvector of h + i beta:  (b, h - a + i beta)  or  (h - dd + i beta, c)
      double p0, q0, p1, q1;
      if (std::abs(b) >= std::abs(c)) {
        p0 = b, q0 = 0.0, p1 = h - a, q1 = beta;
      } else {
        p0 = h - dd, q0 = beta, p1 = c, q1 = 0.0;
      }
      W[0] = p0, W[1] = q0, W[2] = p1, W[3] = q1;
      w[0] = w[1] = h;
      w[2] = beta;
      w[3] = 1.0;
    } else {
      const double r = std::sqrt(disc);
      const double l0 = h + r, l1 = h - r;
      if (std::abs(b) >= std::abs(c)) {
        W[0] = b, W[1] = b, W[2] = l0 - a, W[3] = l1 - a;
      } else {
        W[0] = l0 - dd, W[1] = l1 - dd, W[2] = c, W[3] = c;
      }
      w[0] = l0;
      w[1] = l1;
      w[2] = 0.0;
      w[3] = 2.0;
    }
    const double det = W[0] * W[3] - W[1] * W[2];
    const double nw = std::sqrt(W[0] * W[0] + W[1] * W[1] + W[2] * W[2] + W[3] * W[3]);
    if (!(std::abs(det) > 1e-300) || !(std::abs(det) > 1e-14 * nw * nw)) return false;
    const double Wi[4] = {W[3] / det, -W[1] / det, -W[2] / det, W[0] / det};
    for (int k = 0; k < 4; ++k) {
      w[4 + k] = Wi[k];
      w[8 + k] = W[k];
    }
    const double ni = std::sqrt(Wi[0] * Wi[0] + Wi[1] * Wi[1] + Wi[2] * Wi[2] + Wi[3] * Wi[3]);
    if (max_cond) *max_cond = std::max(*max_cond, nw * ni);
    // Eigenbasis P (columns = eigenvectors), Pinv and eigenvalues, complex.
    using Cx = std::complex<double>;
    Cx P[4], Pi[4], L0, L1;
    if (w[3] == 1.0) {
      // P = W E, E = [[1, 1], [i, -i]];  Pinv = E^{-1} W^{-1}, E^{-1} = 1/2 [[1, -i], [1, i]]
      const Cx I(0.0, 1.0);
      P[0] = W[0] + I * W[1];
      P[1] = W[0] - I * W[1];
      P[2] = W[2] + I * W[3];
      P[3] = W[2] - I * W[3];
      Pi[0] = 0.5 * (Wi[0] - I * Wi[2]);
      Pi[1] = 0.5 * (Wi[1] - I * Wi[3]);
      Pi[2] = 0.5 * (Wi[0] + I * Wi[2]);
      Pi[3] = 0.5 * (Wi[1] + I * Wi[3]);
      L0 = Cx(w[0], w[2]);
      L1 = Cx(w[0], -w[2]);
    } else {
      for (int k = 0; k < 4; ++k) {
        P[k] = W[k];
        Pi[k] = Wi[k];
      }
      L0 = w[0];
      L1 = w[1];
    }
    pr[0] = L0.real(), pr[1] = L0.imag(), pr[2] = L1.real(), pr[3] = L1.imag();
    for (int k = 0; k < 4; ++k) {
      pr[4 + 2 * k] = P[k].real();
      pr[5 + 2 * k] = P[k].imag();
      pr[12 + 2 * k] = Pi[k].real();
      pr[13 + 2 * k] = Pi[k].imag();
    }
  }
  return true;
}

template <typename T>
cudaError_t upload(T** dst, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc(dst, std::max<size_t>(v.size(), 1) * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

// Per-mode tile extents under the kernel caps, honouring n_min / opts.tile.
std::vector<int> choose_tiles(int family, const std::vector<int>& dims, const tsg_opts& o,
                              const tsg::TileCaps caps) {
  (void)family;
  const int d = static_cast<int>(dims.size());
  std::vector<int> b(d);
  for (int m = 0; m < d; ++m) {
    int t = caps.emax;
    if (o.n_min > 0) t = std::min(t, std::max(2, o.n_min));
    if (o.tile[m] > 0) t = std::min(caps.emax, std::max(2, o.tile[m]));
    b[m] = std::min(dims[m], t);
  }
  auto bad = [&]() {
    int64_t E = 1;
    for (int x : b) E *= x;
    if (E > caps.Emax) return true;
    for (int m = 0; m < d; ++m)
      if (E / b[m] > caps.nmax) return true;
    return false;
  };
  while (bad()) {
    int mm = -1;
    for (int m = 0; m < d; ++m)
      if (b[m] > 2 && (mm < 0 || b[m] >= b[mm])) mm = m;
    if (mm < 0) break;
    b[mm] = std::max(2, b[mm] / 2);
  }
  return b;
}

std::vector<int> tile_bounds(int n, int b, const std::vector<int8_t>& code) {
  std::vector<int> bd{0};
  int pos = 0;
  while (pos < n) {
    int end = std::min(pos + b, n);
    if (end < n && code[end] == 2) --end;  // never split a 2x2 block
    if (end <= pos) end = std::min(pos + 2, n);
    bd.push_back(end);
    pos = end;
  }
  return bd;
}

// Eigenvectors of every tile's diagonal block, for the lap3 diagonalised
// tiles.  In the eigenbasis of its 2x2 cells the block is upper triangular
// (That, diagonal lambda; dh tables above), so its eigenvectors Vh are unit
// upper triangular by back substitution:
//   Vh[i][k] = sum_{j >= cend(i)} That[i][j] Vh[j][k] / (lambda_k - lambda_i).
// V = P_tile Vh (columns scaled to unit norm), V^{-1} = Vh^{-1} P_tile^{-1},
// all in long double.  vcond = ||V||_F ||V^{-1}||_F / ext (1 for a normal
// block; inf when two eigenvalues coincide).
// REAL = true: the real block-diagonalising basis instead (see below),
// layout Vr^-1 | Vr (row-major) | alpha | beta, 2 E^2 + 2 E doubles.
template <int E, bool REAL = false>
void tile_eigvecs(std::vector<tsg::TileMode>& tms, const std::vector<double>& dh,
                  const std::vector<double>& pdv, std::vector<double>& vh) {
  using Cx = std::complex<long double>;
  constexpr int EE = E * E, DHS = 2 * EE + 2 * E, VHS = REAL ? 2 * EE + 2 * E : 4 * EE + 2 * E;
  vh.assign(tms.size() * VHS, 0.0);
  for (size_t t = 0; t < tms.size(); ++t) {
    tsg::TileMode& tm = tms[t];
    const int ex = tm.ext;
    const double* o = dh.data() + t * DHS;
    double* out = vh.data() + t * VHS;
    Cx Th[E][E] = {}, lam[E], P[E][E] = {}, Pi[E][E] = {};
    for (int i = 0; i < ex; ++i) {
      lam[i] = Cx(o[2 * EE + i], o[2 * EE + E + i]);
      for (int j = tm.cend[i]; j < ex; ++j) Th[i][j] = Cx(o[i + E * j], o[EE + i + E * j]);
    }
    for (int c = 0; c < tm.nc; ++c) {
      const int r0 = tm.cs[c], z = tm.cz[c];
      if (z == 1) {
        P[r0][r0] = Pi[r0][r0] = 1.0L;
        continue;
      }
      const double* pr = pdv.data() + static_cast<size_t>(tm.start + r0) * tsg::kPStride;
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
          P[r0 + a][r0 + b] = Cx(pr[4 + (a * 2 + b) * 2], pr[5 + (a * 2 + b) * 2]);
          Pi[r0 + a][r0 + b] = Cx(pr[12 + (a * 2 + b) * 2], pr[13 + (a * 2 + b) * 2]);
        }
    }
    Cx Vh[E][E] = {}, W[E][E] = {};
    bool ok = true;
    for (int k = 0; k < ex && ok; ++k) {
      Vh[k][k] = 1.0L;
      for (int i = k - 1; i >= 0; --i) {
        Cx s = 0.0L;
        for (int j = tm.cend[i]; j <= k; ++j) s += Th[i][j] * Vh[j][k];
        const Cx dl = lam[k] - lam[i];
        if (std::abs(s) == 0.0L) continue;
        if (std::abs(dl) == 0.0L) {
          ok = false;
          break;
        }
        Vh[i][k] = s / dl;
      }
    }
    for (int c = 0; c < ex && ok; ++c) {  // W = Vh^{-1}
      W[c][c] = 1.0L;
      for (int i = c - 1; i >= 0; --i) {
        Cx s = 0.0L;
        for (int j = i + 1; j <= c; ++j) s += Vh[i][j] * W[j][c];
        W[i][c] = -s;
      }
    }
    Cx V[E][E] = {}, Vi[E][E] = {};
    long double nv = 0, ni = 0;
    if (ok) {
      for (int i = 0; i < ex; ++i)
        for (int k = 0; k < ex; ++k)
          for (int j = 0; j < ex; ++j) {
            V[i][k] += P[i][j] * Vh[j][k];
            Vi[i][k] += W[i][j] * Pi[j][k];
          }
      for (int k = 0; k < ex; ++k) {  // unit columns of V, matching rows of V^{-1}
        long double cn = 0;
        for (int i = 0; i < ex; ++i) cn += std::norm(V[i][k]);
        cn = std::sqrt(cn);
        for (int i = 0; i < ex; ++i) {
          V[i][k] /= cn;
          Vi[k][i] *= cn;
        }
      }
      for (int i = 0; i < ex; ++i)
        for (int k = 0; k < ex; ++k) {
          nv += std::norm(V[i][k]);
          ni += std::norm(Vi[i][k]);
        }
    }
    const long double vc = ok ? std::sqrt(nv * ni) / ex : 0.0L;
    tm.vcond = ok && std::isfinite(static_cast<double>(vc)) ? static_cast<float>(vc)
                                                           : std::numeric_limits<float>::infinity();
    if constexpr (REAL) {
      // Real block-diagonalising basis: a real eigenvalue keeps its (phase-
      // normalised, real) eigenvector; a complex pair alpha +- i beta of cell
      // rows (r, r+1) takes [Re v_r, Im v_r], for which
      // D [Re v, Im v] = [Re v, Im v] [[alpha, beta], [-beta, alpha]].
      long double Vr[E][E] = {}, Vri[E][E] = {};
      bool okr = ok;
      for (int c = 0; c < tm.nc && okr; ++c) {
        const int r0 = tm.cs[c];
        if (tm.cz[c] == 1) {
          int im = 0;
          for (int i = 1; i < ex; ++i)
            if (std::abs(V[i][r0]) > std::abs(V[im][r0])) im = i;
          const Cx ph = V[im][r0] / std::abs(V[im][r0]);
          for (int i = 0; i < ex; ++i) Vr[i][r0] = (V[i][r0] / ph).real();
        } else {
          for (int i = 0; i < ex; ++i) {
            Vr[i][r0] = V[i][r0].real();
            Vr[i][r0 + 1] = V[i][r0].imag();
          }
        }
      }
      // Vri = Vr^{-1} (Gauss-Jordan, partial pivoting, long double)
      if (okr) {
        long double Aug[E][2 * E] = {};
        for (int i = 0; i < ex; ++i) {
          for (int k = 0; k < ex; ++k) Aug[i][k] = Vr[i][k];
          Aug[i][ex + i] = 1.0L;
        }
        for (int col = 0; col < ex && okr; ++col) {
          int pv = col;
          for (int i = col + 1; i < ex; ++i)
            if (std::fabs(Aug[i][col]) > std::fabs(Aug[pv][col])) pv = i;
          if (Aug[pv][col] == 0.0L) {
            okr = false;
            break;
          }
          if (pv != col)
            for (int k = 0; k < 2 * ex; ++k) std::swap(Aug[pv][k], Aug[col][k]);
          const long double inv = 1.0L / Aug[col][col];
          for (int k = 0; k < 2 * ex; ++k) Aug[col][k] *= inv;
          for (int i = 0; i < ex; ++i) {
            if (i == col || Aug[i][col] == 0.0L) continue;
            const long double f = Aug[i][col];
            for (int k = 0; k < 2 * ex; ++k) Aug[i][k] -= f * Aug[col][k];
          }
        }
        for (int i = 0; i < ex; ++i)
          for (int k = 0; k < ex; ++k) Vri[i][k] = Aug[i][ex + k];
      }
      long double nr = 0, nri = 0;
      for (int i = 0; i < ex; ++i)
        for (int k = 0; k < ex; ++k) {
          nr += Vr[i][k] * Vr[i][k];
          nri += Vri[i][k] * Vri[i][k];
        }
      const long double vcr = okr ? std::sqrt(nr * nri) / ex : 0.0L;
      tm.vcond = okr && std::isfinite(static_cast<double>(vcr)) ? static_cast<float>(vcr)
                                                               : std::numeric_limits<float>::infinity();
      for (int i = 0; i < E; ++i) {
        for (int k = 0; k < E; ++k) {
          const bool in = i < ex && k < ex;
          out[i * E + k] = in ? static_cast<double>(Vri[i][k]) : (i == k ? 1.0 : 0.0);
          out[EE + i * E + k] = in ? static_cast<double>(Vr[i][k]) : (i == k ? 1.0 : 0.0);
        }
        out[2 * EE + i] = i < ex ? static_cast<double>(lam[i].real()) : 1.0;
        out[2 * EE + E + i] = i < ex ? static_cast<double>(lam[i].imag()) : 0.0;
      }
      continue;
    }
    for (int i = 0; i < E; ++i) {
      for (int k = 0; k < E; ++k) {
        const bool in = i < ex && k < ex;
        const Cx vi = in ? Vi[i][k] : Cx(i == k ? 1.0L : 0.0L);
        const Cx v = in ? V[i][k] : Cx(i == k ? 1.0L : 0.0L);
        out[i * E + k] = static_cast<double>(vi.real());
        out[EE + i * E + k] = static_cast<double>(vi.imag());
        out[2 * EE + i * E + k] = static_cast<double>(v.real());
        out[3 * EE + i * E + k] = static_cast<double>(v.imag());
      }
      out[4 * EE + i] = i < ex ? static_cast<double>(lam[i].real()) : 1.0;
      out[4 * EE + E + i] = i < ex ? static_cast<double>(lam[i].imag()) : 0.0;
    }
  }
}

int try_decouple(tsg_plan* pl, const double* const* T, const double* const* U, const double* Tc);
int enqueue(tsg_plan* pl, const double* in, double* out, cudaStream_t st, bool timing);

}  // namespace

namespace tsg_impl {
std::vector<int> tile_bounds_of(const double* T, int n, int b) {
  return tile_bounds(n, b, block_codes(T, n));
}
}  // namespace tsg_impl

PlanKnobs PlanKnobs::from_env() {
  PlanKnobs k;
  const char* g = std::getenv("TSG_GATE");
  k.serial = g && std::atoi(g) == 0;
  const char* sc = std::getenv("TSG_SCHAIN");
  k.schain_off = sc && std::atoi(sc) == 0;
  k.verbose = std::getenv("TSG_VERBOSE") != nullptr;
#ifdef TSG_DEVTOOLS
  k.trace = std::getenv("TSG_TRACE") != nullptr;
  k.prof = std::getenv("TSG_PROF") != nullptr;
  k.dbg_fdone = std::getenv("TSG_DBG_FDONE") != nullptr;
  if (const char* e = std::getenv("TSG_DBG")) k.dbg = std::atoi(e);
#endif
  return k;
}

// All-mode transform in -> target (definition below)
cudaError_t transform_all(tsg_plan* pl, const double* in, double* target, double* other, bool fwd,
                          cudaStream_t st, const tsg::GemmArgs* gate0 = nullptr,
                          cudaEvent_t after0 = nullptr, int i_lo = 0, int i_hi = -1,
                          const tsg::GemmArgs* last = nullptr);

extern "C" {

int tsg_abi_version(void) { return 1; }

void tsg_default_opts(tsg_opts* o) {
  std::memset(o, 0, sizeof(*o));
  o->free_mode = -1;
}

int tsg_create(int n_gpus, const int* device_ids, tsg_ctx** out) {
  if (!out) return TSG_EINVAL;
  *out = nullptr;
  if (n_gpus != 1) return TSG_EINVAL;  // slab sharding: one process per GPU
  auto* ctx = new tsg_ctx();
  ctx->device = device_ids ? device_ids[0] : 0;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  for (int i = 0; i < 8 && e == cudaSuccess; ++i) e = cudaEventCreate(&ctx->ev[i]);
  if (e != cudaSuccess) {
    delete ctx;
    return TSG_ECUDA;
  }
  *out = ctx;
  return TSG_OK;
}

void tsg_destroy(tsg_ctx* ctx) {
  if (!ctx) return;
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* tsg_last_error(const tsg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void* tsg_ctx_stream(const tsg_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int tsg_plan_create(tsg_ctx* ctx, int family, int d, const int* dims, const double* const* T,
                    const double* const* U, const double* Tc, const double* Z, int reduced_only,
                    const tsg_opts* opts, tsg_plan** out) {
  if (!ctx || !out) return TSG_EINVAL;
  *out = nullptr;
  tsg_opts o;
  tsg_default_opts(&o);
  if (opts) o = *opts;
  if (d < 2 || d > 6) return fail(ctx, TSG_EDIM, "order d must be in [2, 6]");
  if (family == 1 && !Tc) return fail(ctx, TSG_EDIM, "gsylv needs the Tc factor");
  for (int m = 0; m < d; ++m) {
    if (dims[m] <= 0) return fail(ctx, TSG_EDIM, "dimensions must be positive");
    if (!T[m]) return fail(ctx, TSG_EDIM, "missing coefficient");
    if (!reduced_only && !U[m] && !((o.skip_transform_mask >> m) & 1))
      return fail(ctx, TSG_EDIM, "missing orthogonal factor");
    if (!quasi_upper(T[m], dims[m]))
      return fail(ctx, TSG_EDIM,
                  "coefficient " + std::to_string(m) + " must be upper quasi-triangular");
  }
  if (family == 1) {
    if (!upper(Tc, dims[0])) return fail(ctx, TSG_EDIM, "C must be upper triangular");
    if (!reduced_only && !Z) return fail(ctx, TSG_EDIM, "missing Z factor");
  }
  TSG_CU(cudaSetDevice(ctx->device));
  auto pl = std::make_unique<tsg_plan>();
  pl->knobs = PlanKnobs::from_env();
  pl->skip_mask = o.skip_transform_mask & ((1 << d) - 1);
  pl->force_f = o.free_mode;
  if (pl->force_f < 0)
    if (const char* e = std::getenv("TSG_DECOUPLE_F")) pl->force_f = std::atoi(e);  // tuning knob
  pl->ctx = ctx;
  pl->family = family;
  pl->d = d;
  pl->reduced_only = reduced_only;
  pl->dims.assign(dims, dims + d);
  pl->stride.resize(d);
  int64_t s = 1;
  for (int m = 0; m < d; ++m) {
    pl->stride[m] = s;
    s *= dims[m];
  }
  pl->N = s;
  pl->T.resize(d);
  pl->Fwd.resize(d);
  pl->FwdT.resize(d);
  pl->Bwd.resize(d);
  pl->BwdT.resize(d);
  pl->eig.resize(d);
  pl->pdat.resize(d);
  pl->dhat.resize(d);
  pl->vhat.resize(d);
  std::vector<std::vector<double>> pdvs(d), nfs(d);
  pl->tmode.assign(d, nullptr);
  pl->bnd.assign(d, nullptr);
  pl->rowtile.assign(d, nullptr);

  double scale = 0;
  std::vector<std::vector<int8_t>> codes(d);
  for (int m = 0; m < d; ++m) {
    const int n = dims[m];
    const size_t nn = static_cast<size_t>(n) * n;
    TSG_CU(upload_mat(pl->T[m], T[m], nn));
    codes[m] = block_codes(T[m], n);
    std::vector<double> nf, pdv;
    if (!normal_form(T[m], n, codes[m], nf, pdv, &pl->max_cond))
      return fail(ctx, TSG_EDIM, "coefficient " + std::to_string(m) +
                                     " has a defective 2x2 diagonal block (equal real eigenvalues)");
    TSG_CU(upload_mat(pl->eig[m], nf.data(), nf.size()));
    TSG_CU(upload_mat(pl->pdat[m], pdv.data(), pdv.size()));
    pdvs[m] = pdv;
    nfs[m] = nf;
    scale += fro(T[m], nn);
    if (!reduced_only && !((pl->skip_mask >> m) & 1)) {
      // forward: A = U^T (mode 0), At = U (m > 0); back: A = U, At = U^T.
      // gsylv mode 0: forward Q^T, back Z.
      const double* bk = (family == 1 && m == 0) ? Z : U[m];
      const std::vector<double> ut = transpose(U[m], n), bt = transpose(bk, n);
      TSG_CU(upload_mat(pl->Fwd[m], ut.data(), nn));
      TSG_CU(upload_mat(pl->FwdT[m], U[m], nn));
      TSG_CU(upload_mat(pl->Bwd[m], bk, nn));
      TSG_CU(upload_mat(pl->BwdT[m], bt.data(), nn));
    }
  }
  if (family == 1) {
    const size_t nn = static_cast<size_t>(dims[0]) * dims[0];
    TSG_CU(upload_mat(pl->Tc, Tc, nn));
    scale += fro(Tc, nn);
  }
  pl->tiny = 0.5 * std::numeric_limits<double>::epsilon() * scale;
  {
    const int rc = try_decouple(pl.get(), T, U, Tc);
    if (rc != TSG_OK) return rc;
  }
  if (pl->decoupled) {
    TSG_CU(cudaMalloc(&pl->flags, sizeof(int)));
    TSG_CU(cudaMalloc(&pl->counter, 2 * sizeof(int)));
    TSG_CU(cudaMemset(pl->counter, 0x7f, 2 * sizeof(int)));  // status word: kNoStatus
    pl->ntiles = 1;
    static const bool small_on = [] {
      const char* e = std::getenv("TSG_SMALLMODES");
      return !e || std::atoi(e) != 0;
    }();
    const bool two_gemm = !(small_on && (tsg::small_mode_ok(dims[0]) || tsg::small_mode_ok(dims[1])));
    if (d >= 3 && two_gemm && pl->N / (static_cast<int64_t>(dims[0]) * dims[1]) > 1) {
      int bm = 0, bn = 0;
      const int64_t Q0 = pl->N / dims[0];
      tsg::gemm_tile_shape(dims[0], static_cast<int>(Q0), &bm, &bn);
      if (bm > 0 && bn > 0 && Q0 < INT_MAX) {
        pl->s_tm = (dims[0] + bm - 1) / bm;
        pl->s_bn = bn;
        pl->sdone_n = pl->s_tm * static_cast<int>((Q0 + bn - 1) / bn);
      }
    }
    TSG_CU(tsg::gemm_prepare());
    pl->aux_n = 2 * static_cast<int64_t>(pl->sdone_n);
    if (pl->aux_n > 0) {
      TSG_CU(cudaMalloc(&pl->aux, pl->aux_n * sizeof(int)));
      pl->sdone[0] = pl->aux;
      pl->sdone[1] = pl->aux + pl->sdone_n;
    }
    double sn = 0, snm1 = 0;
    for (int m = 0; m < d; ++m) {
      sn += dims[m];
      snm1 += dims[m] - 1;
    }
    const double Nd = static_cast<double>(pl->N);
    pl->flops_alg = (family == 0 ? Nd * snm1 : Nd * ((dims[0] - 1) + sn)) + 4.0 * Nd * sn;
    // complex back substitution: n_f^2 real FMA per pair of real fibres
    // (gsylv: two triangular factors, S and Tc)
    pl->flops_exec = (family == 0 ? 1.0 : 2.0) * Nd * dims[pl->dec_f] + 4.0 * Nd * sn;
    TSG_CU(pl->w1.ensure(pl->N));
    TSG_CU(pl->w2.ensure(pl->N));
    *out = pl.release();
    return TSG_OK;
  }
  // Closed-form base cells lose ~eps*cond(V); refine when some block's
  // eigenbasis is poorly conditioned (rare for LAPACK-standardised blocks).
  pl->refine = pl->max_cond > 1e3 ? 1 : 0;
  if (const char* e = std::getenv("TSG_REFINE")) pl->refine = std::atoi(e);

  // Kernel choice: the fast Laplace path needs well-conditioned eigenbases
  // (no refinement step); gsylv and the rest use the generic kernel.
  pl->fast = (family == 0 && !pl->refine) ? (d == 3 ? 3 : 1) : 0;
  if (const char* e = std::getenv("TSG_FAST")) pl->fast = std::atoi(e);
  if (pl->fast == 3 && d != 3) pl->fast = 1;
  if (family != 0) pl->fast = 0;
  pl->lt3 = 3;
  if (const char* e = std::getenv("TSG_LT")) pl->lt3 = std::atoi(e) == 4 ? 4 : 3;
  // Tiles (host tables first; the 16^3 TMA kernel is taken when every tile's
  // eigenvector bases are well conditioned, else the 8^3 kernel).
  struct ModeTables {
    std::vector<int> bd;
    std::vector<tsg::TileMode> tms;
    std::vector<double> dh, vh;
    float maxvc = 0.0f;
  };
  std::vector<ModeTables> mts(d);
  auto build_mode = [&](int m, int lt, bool diag16) -> int {
    ModeTables& mt = mts[m];
    mt = ModeTables{};
    mt.bd = tile_bounds(dims[m], pl->tile_ext[m], codes[m]);
    const int ntm = static_cast<int>(mt.bd.size()) - 1;
    mt.tms.resize(ntm);
    for (int t = 0; t < ntm; ++t) {
      tsg::TileMode& tmd = mt.tms[t];
      std::memset(&tmd, 0, sizeof(tmd));
      tmd.start = mt.bd[t];
      const int ex = mt.bd[t + 1] - mt.bd[t];
      if (ex > 255) return fail(ctx, TSG_EDIM, "tile extent too large");
      tmd.ext = static_cast<unsigned char>(ex);
      int nc = 0;
      for (int r = 0; r < ex;) {
        const int sz = codes[m][tmd.start + r] == 1 ? 2 : 1;
        if (nc >= tsg::kMaxCells) return fail(ctx, TSG_EDIM, "too many Schur cells in a tile");
        tmd.cs[nc] = static_cast<unsigned char>(r);
        tmd.cz[nc] = static_cast<unsigned char>(sz);
        if (sz == 2) tmd.pair = 1;
        for (int q = r; q < r + sz; ++q) {
          tmd.cellof[q] = static_cast<unsigned char>(nc);
          tmd.cend[q] = static_cast<unsigned char>(r + sz);
        }
        tmd.cplx[r] = sz == 2 ? 1 : 0;
        if (sz == 2 && nfs[m][static_cast<size_t>(tmd.start + r) * tsg::kEigStride + 3] == 1.0) {
          tmd.ckind[r] = 1;
          tmd.ckind[r + 1] = 2;
        }
        ++nc;
        r += sz;
      }
      tmd.nc = static_cast<unsigned char>(nc);
      tmd.far_lo = t + 3 < ntm ? mt.bd[t + 3] : dims[m];
    }
    if (pl->fast == 3 || pl->fast == 5 || pl->fast == 6) {
      // Eigenbasis diagonal block of every tile index along mode m:
      // That[i][j] = sum Pinv_blk(i)[i,a] T[a,b] P_blk(j)[b,j] for j beyond
      // i's cell (0 elsewhere), then lambda_i; layout of solve_lap3 (DHS).
      using Cx = std::complex<double>;
      const int E = 1 << lt, EE = E * E, DHS = 2 * EE + 2 * E;
      std::vector<double>& dh = mt.dh;
      dh.assign(static_cast<size_t>(ntm) * DHS, 0.0);
      const int n = dims[m];
      auto Pget = [&](int row0, int r, int c, int which) {  // which 4: P, 12: Pinv
        const double* pr = pdvs[m].data() + static_cast<size_t>(row0) * tsg::kPStride + which;
        return Cx(pr[(r * 2 + c) * 2], pr[(r * 2 + c) * 2 + 1]);
      };
      for (int t = 0; t < ntm; ++t) {
        const tsg::TileMode& tmd = mt.tms[t];
        double* o = dh.data() + static_cast<size_t>(t) * DHS;
        for (int i = 0; i < tmd.ext; ++i) {
          const int ci = tmd.cellof[i], I0 = tmd.cs[ci], Iz = tmd.cz[ci];
          for (int j = tmd.cend[i]; j < tmd.ext; ++j) {
            const int cj = tmd.cellof[j], J0 = tmd.cs[cj], Jz = tmd.cz[cj];
            Cx acc(0.0, 0.0);
            for (int aa = 0; aa < Iz; ++aa)
              for (int bb = 0; bb < Jz; ++bb) {
                const double dv = at(T[m], n, tmd.start + I0 + aa, tmd.start + J0 + bb);
                const Cx w = Iz == 2 ? Pget(tmd.start + I0, i - I0, aa, 12) : Cx(1.0, 0.0);
                const Cx v = Jz == 2 ? Pget(tmd.start + J0, bb, j - J0, 4) : Cx(1.0, 0.0);
                acc += w * dv * v;
              }
            o[i + E * j] = acc.real();
            o[EE + i + E * j] = acc.imag();
          }
          const double* pr = pdvs[m].data() + static_cast<size_t>(tmd.start + I0) * tsg::kPStride;
          o[2 * EE + i] = pr[(i - I0) * 2];
          o[2 * EE + E + i] = pr[(i - I0) * 2 + 1];
        }
      }
      if (lt == 3) tile_eigvecs<8>(mt.tms, dh, pdvs[m], mt.vh);
      else if (diag16) tile_eigvecs<16, true>(mt.tms, dh, pdvs[m], mt.vh);
      for (const auto& tm : mt.tms) mt.maxvc = std::max(mt.maxvc, tm.vcond);
    }
    return TSG_OK;
  };
  const char* e16 = std::getenv("TSG_LAP16");
  const bool want16 = pl->fast == 3 && d == 3 && !tsg_impl::g_force_lap3 && !std::getenv("TSG_LT") &&
                      (e16 ? std::atoi(e16) != 0
                           : (dims[0] >= 64 && dims[1] >= 64 && dims[2] >= 64 && pl->N >= (int64_t{1} << 23))) &&
                      dims[0] % 2 == 0 &&  // TMA: 16-byte row strides
                      dims[0] <= 1024 && dims[1] <= 1024 && dims[2] <= 1024;  // per-tile chunk list
  if (want16) {
    pl->tile_ext = choose_tiles(family, pl->dims, o, tsg::solve_lap16_caps());
    double prod = 1.0;
    for (int m = 0; m < d; ++m) {
      const int rc = build_mode(m, 4, true);
      if (rc != TSG_OK) return rc;
      prod *= mts[m].maxvc;
    }
    if (prod <= tsg::kDiagCond) {
      pl->use16 = true;
      pl->lt3 = 4;
    }
  }
  // order >= 4 Laplace: the diagonalised small-tile kernel when its padded
  // tiles fit (<= 512 unknowns) and every tile's bases are well conditioned
  const char* ed = std::getenv("TSG_LAPD");
  if (!pl->use16 && pl->fast == 1 && d >= 4 && (ed ? std::atoi(ed) != 0 : true)) {
    pl->fast = 5;
    pl->tile_ext = choose_tiles(family, pl->dims, o, tsg::solve_lapd_caps());
    double prod = 1.0;
    int lsum = 0;
    pl->tlog.assign(d, 0);
    pl->tsh.assign(d, 0);
    for (int m = 0; m < d; ++m) {
      const int rc = build_mode(m, 3, false);
      if (rc != TSG_OK) return rc;
      prod *= mts[m].maxvc;
      int mx = 1;
      for (const auto& tm : mts[m].tms) mx = std::max(mx, static_cast<int>(tm.ext));
      int lg = 0;
      while ((1 << lg) < mx) ++lg;
      pl->tsh[m] = lsum;
      pl->tlog[m] = lg;
      lsum += lg;
    }
    if (!(prod <= tsg::kDiagCond) || (1 << lsum) > tsg::solve_lapd_caps().Emax) pl->fast = 1;
  }
  // gsylv d = 3..5: the small-tile kernel when the tail tiles' bases are
  // well conditioned (mode 0 is solved by back substitution, no basis)
  const char* eg = std::getenv("TSG_GSYD");
  if (family == 1 && d >= 3 && d <= 5 && (eg ? std::atoi(eg) != 0 : true)) {
    pl->fast = 6;
    pl->tile_ext = choose_tiles(family, pl->dims, o, tsg::solve_gsyd_caps());
    double prod = 1.0;
    int lsum = 0;
    pl->tlog.assign(d, 0);
    pl->tsh.assign(d, 0);
    for (int m = 0; m < d; ++m) {
      const int rc = build_mode(m, 3, false);
      if (rc != TSG_OK) return rc;
      if (m > 0) prod *= mts[m].maxvc;
      int mx = 1;
      for (const auto& tm : mts[m].tms) mx = std::max(mx, static_cast<int>(tm.ext));
      int lg = 0;
      while ((1 << lg) < mx) ++lg;
      pl->tsh[m] = lsum;
      pl->tlog[m] = lg;
      lsum += lg;
    }
    if (!(prod <= tsg::kDiagCond) || lsum > 9) pl->fast = 0;
  }
  if (!pl->use16 && pl->fast != 5 && pl->fast != 6) {
    pl->tile_ext = choose_tiles(family, pl->dims, o,
                                pl->fast == 3 ? tsg::solve_lap3_caps(pl->lt3)
                                              : (pl->fast ? tsg::solve_lap_caps(d) : tsg::solve_caps(family, d)));
    for (int m = 0; m < d; ++m) {
      const int rc = build_mode(m, pl->lt3, false);
      if (rc != TSG_OK) return rc;
    }
  }
  pl->ntiles_mode.resize(d);
  pl->ntiles = 1;
  std::vector<std::vector<int>> bds(d);
  for (int m = 0; m < d; ++m) {
    bds[m] = mts[m].bd;
    pl->ntiles_mode[m] = static_cast<int>(bds[m].size()) - 1;
    pl->ntiles *= pl->ntiles_mode[m];
    TSG_CU(upload(&pl->bnd[m], bds[m]));
    {
      std::vector<int> rt(dims[m], 0);
      for (int t = 0; t + 1 < static_cast<int>(bds[m].size()); ++t)
        for (int i = bds[m][t]; i < bds[m][t + 1]; ++i) rt[i] = t;
      TSG_CU(upload(&pl->rowtile[m], rt));
    }
    if (!mts[m].dh.empty()) TSG_CU(upload_mat(pl->dhat[m], mts[m].dh.data(), mts[m].dh.size()));
    if (!mts[m].vh.empty()) TSG_CU(upload_mat(pl->vhat[m], mts[m].vh.data(), mts[m].vh.size()));
    TSG_CU(upload(&pl->tmode[m], mts[m].tms));
  }
  pl->bds_h = bds;
  if (pl->ntiles > INT_MAX / 2) return fail(ctx, TSG_EDIM, "too many tiles");
  for (int m = 0; m < d; ++m)
    if (pl->ntiles_mode[m] > 1024) return fail(ctx, TSG_EDIM, "more than 1024 tiles along a mode");
  // Topological order: hyperplane sum_m t_m descending.
  {
    std::vector<int> hp(pl->ntiles), ord(pl->ntiles);
    for (int64_t t = 0; t < pl->ntiles; ++t) {
      int64_t r = t;
      int h = 0;
      for (int m = 0; m < d; ++m) {
        h += static_cast<int>(r % pl->ntiles_mode[m]);
        r /= pl->ntiles_mode[m];
      }
      hp[t] = h;
      ord[t] = static_cast<int>(t);
    }
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return hp[x] > hp[y]; });
    TSG_CU(upload(&pl->order, ord));
    pl->order_h = ord;
    std::vector<unsigned long long> oc(pl->ntiles);
    for (int64_t q = 0; q < pl->ntiles; ++q) {
      int64_t r = ord[q];
      unsigned long long pk = 0;
      for (int m = 0; m < d; ++m) {
        pk |= static_cast<unsigned long long>(r % pl->ntiles_mode[m]) << (10 * m);
        r /= pl->ntiles_mode[m];
      }
      oc[q] = pk;
    }
    TSG_CU(upload(&pl->ocoord, oc));
  }
  TSG_CU(cudaMalloc(&pl->flags, pl->ntiles * sizeof(int)));
  TSG_CU(cudaMalloc(&pl->counter, 2 * sizeof(int)));
  TSG_CU(cudaMemset(pl->counter, 0x7f, 2 * sizeof(int)));  // status word: kNoStatus

  // Gate of the overlapped back transform (Laplace tile kernels whose first
  // back pass is a mode-0 GEMM).  Tile (0, t_1, ..) released implies every
  // tile (t_0, t_1, ..) is: each waits on its successor along mode 0.
  {
    static const bool small_on = [] {
      const char* e = std::getenv("TSG_SMALLMODES");
      return !e || std::atoi(e) != 0;
    }();
    const bool first_gemm = !(small_on && tsg::small_mode_ok(dims[0]));
    if (family == 0 && !pl->reduced_only && d >= 2 && first_gemm &&
        (pl->use16 || pl->fast == 3 || pl->fast == 5)) {
      const int64_t Q = pl->N / dims[0];
      const int64_t G = (Q + tsg::kWaitCols - 1) / tsg::kWaitCols;
      std::vector<std::vector<int>> t_of(d);
      for (int m = 1; m < d; ++m) {
        t_of[m].resize(dims[m]);
        for (int t = 0; t < pl->ntiles_mode[m]; ++t)
          for (int i = bds[m][t]; i < bds[m][t + 1]; ++i) t_of[m][i] = t;
      }
      std::vector<int64_t> mul(d, 1);
      for (int m = 1; m < d; ++m) mul[m] = mul[m - 1] * pl->ntiles_mode[m - 1];
      std::vector<int> off(G + 1, 0), ids, grp;
      std::vector<int> idx(d, 0);  // multi-index over modes 1..d-1 (mode 1 fastest)
      for (int64_t gi = 0; gi < G; ++gi) {
        grp.clear();
        const int64_t c1 = std::min<int64_t>(Q, (gi + 1) * tsg::kWaitCols);
        for (int64_t c = gi * tsg::kWaitCols; c < c1; ++c) {
          int64_t id = 0;
          for (int m = 1; m < d; ++m) id += t_of[m][idx[m]] * mul[m];
          if (grp.empty() || grp.back() != id) grp.push_back(static_cast<int>(id));
          for (int m = 1; m < d; ++m) {
            if (++idx[m] < dims[m]) break;
            idx[m] = 0;
          }
        }
        std::sort(grp.begin(), grp.end());
        grp.erase(std::unique(grp.begin(), grp.end()), grp.end());
        ids.insert(ids.end(), grp.begin(), grp.end());
        off[gi + 1] = static_cast<int>(ids.size());
      }
      TSG_CU(upload(&pl->gate_off, off));
      TSG_CU(upload(&pl->gate_ids, ids));
      pl->gate_groups = static_cast<int>(G);
    }
    // Slab chain mode 0 -> mode 1 (both GEMM passes, mode 1 batched)
    const bool two_gemm = !(small_on && (tsg::small_mode_ok(dims[0]) || tsg::small_mode_ok(dims[1])));
    if (!pl->reduced_only && d >= 3 && two_gemm && pl->N / (static_cast<int64_t>(dims[0]) * dims[1]) > 1) {
      int bm = 0, bn = 0;
      const int64_t Q0 = pl->N / dims[0];
      tsg::gemm_tile_shape(dims[0], static_cast<int>(Q0), &bm, &bn);
      if (bm > 0 && bn > 0 && Q0 < INT_MAX) {
        pl->s_tm = (dims[0] + bm - 1) / bm;
        pl->s_bn = bn;
        pl->sdone_n = pl->s_tm * static_cast<int>((Q0 + bn - 1) / bn);
      }
    }
    TSG_CU(tsg::gemm_prepare());  // kernel attributes before any launch chain (see gemm.cu)
    // Trailing cube (TSG_CUBE = tiles per mode, default 6, 0 = off; TSG_CUBE_GRID CTAs, default 16)
    {
      const char* ce = std::getenv("TSG_CUBE");
      const int L1 = ce ? std::atoi(ce) : 6;
      const char* cg = std::getenv("TSG_CUBE_GRID");
      // three GEMM forward passes (enqueue splits them 2 + 1 around the cube grid)
      bool ok = L1 > 0 && family == 0 && !pl->reduced_only && d == 3 && pl->use16 && tsg::lap16_decoupled() &&
                !(small_on && (tsg::small_mode_ok(dims[0]) || tsg::small_mode_ok(dims[1]) ||
                               tsg::small_mode_ok(dims[2])));
      for (int m = 0; ok && m < d; ++m) ok = pl->ntiles_mode[m] >= L1 + 3;
      int bm = 0, bn = 0;
      if (ok) tsg::gemm_tile_shape(dims[0] * dims[1], dims[2], &bm, &bn);
      int nsm = 0;
      if (ok) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
      if (ok && bm > 0 && bn > 0 && nsm >= 4 * (cg ? std::max(1, std::atoi(cg)) : 16)) {
        pl->cube = L1;
        pl->cube_grid = cg ? std::max(1, std::atoi(cg)) : 16;
        pl->fg_bm = bm;
        pl->fg_bn = bn;
        pl->fg_tm = (dims[0] * dims[1] + bm - 1) / bm;
        pl->fdone_n = pl->fg_tm * ((dims[2] + bn - 1) / bn);
        std::vector<int> o1, o2;
        std::vector<unsigned long long> c1, c2;
        for (int64_t q = 0; q < pl->ntiles; ++q) {
          int64_t r = pl->order_h[q];
          bool in = true;
          unsigned long long pk = 0;
          for (int m = 0; m < d; ++m) {
            const int t = static_cast<int>(r % pl->ntiles_mode[m]);
            r /= pl->ntiles_mode[m];
            in = in && t >= pl->ntiles_mode[m] - L1;
            pk |= static_cast<unsigned long long>(t) << (10 * m);
          }
          (in ? o1 : o2).push_back(pl->order_h[q]);
          (in ? c1 : c2).push_back(pk);
        }
        TSG_CU(upload(&pl->order1, o1));
        TSG_CU(upload(&pl->order2, o2));
        TSG_CU(upload(&pl->ocoord1, c1));
        TSG_CU(upload(&pl->ocoord2, c2));
        pl->ntiles1 = static_cast<int64_t>(o1.size());
        pl->ntiles2 = static_cast<int64_t>(o2.size());
      }
    }
    // one allocation for the per-solve auxiliary flags (reset with the tile flags)
    pl->aux_n = 2 * static_cast<int64_t>(pl->sdone_n) + pl->fdone_n + (pl->cube ? 1 : 0);
    if (pl->aux_n > 0) {
      TSG_CU(cudaMalloc(&pl->aux, pl->aux_n * sizeof(int)));
      if (pl->sdone_n) {
        pl->sdone[0] = pl->aux;
        pl->sdone[1] = pl->aux + pl->sdone_n;
      }
      if (pl->cube) pl->fdone = pl->aux + 2 * static_cast<int64_t>(pl->sdone_n);
    }
  }

  // Executed FLOP of the solve: left-looking updates per tile and pass.
  {
    double fe = 0;
    const int npass_extra = family == 1 ? 1 : 0;  // gsylv mode 0 has two sources
    for (int m = 0; m < d; ++m) {
      // sum over tiles of 2 * E_t * (extent of later tiles along m)
      // = 2 * sum_{t_m} e_{t_m} * (n_m - bnd[t_m+1]) * prod_{v != m} n_v
      double acc = 0;
      for (int t = 0; t < pl->ntiles_mode[m]; ++t)
        acc += static_cast<double>(bds[m][t + 1] - bds[m][t]) * (dims[m] - bds[m][t + 1]);
      fe += 2.0 * acc * (static_cast<double>(pl->N) / dims[m]) * (m == 0 ? 1 + npass_extra : 1);
      // in-tile part: each strictly-upper coefficient inside a tile once
      double in = 0;
      for (int t = 0; t < pl->ntiles_mode[m]; ++t) {
        const double e = bds[m][t + 1] - bds[m][t];
        in += e * (e - 1) / 2;
      }
      fe += 2.0 * in * (static_cast<double>(pl->N) / dims[m]) * (m == 0 ? 1 + npass_extra : 1);
    }
    double sn = 0, snm1 = 0;
    for (int m = 0; m < d; ++m) {
      sn += dims[m];
      snm1 += dims[m] - 1;
    }
    const double Nd = static_cast<double>(pl->N);
    double falg_solve = family == 0 ? Nd * snm1 : Nd * ((dims[0] - 1) + (sn));
    pl->flops_alg = falg_solve + (reduced_only ? 0.0 : 4.0 * Nd * sn);
    pl->flops_exec = fe + (reduced_only ? 0.0 : 4.0 * Nd * sn);
  }

  // Work buffers.
  TSG_CU(pl->w1.ensure(pl->N));
  if (!reduced_only) TSG_CU(pl->w2.ensure(pl->N));
  if (family == 1) {
    pl->wchain.resize(d);
    for (int m = 1; m < d; ++m) TSG_CU(pl->wchain[m].ensure(pl->N));
  }
  *out = pl.release();
  return TSG_OK;
}

void tsg_plan_destroy(tsg_plan* plan) { delete plan; }

int tsg_plan_info(const tsg_plan* pl, int64_t* n_tiles, int* tile_extents, double* flops_alg) {
  if (!pl) return TSG_EINVAL;
  if (n_tiles) *n_tiles = pl->ntiles;
  if (tile_extents)
    for (int m = 0; m < pl->d; ++m) tile_extents[m] = pl->tile_ext[m];
  if (flops_alg) *flops_alg = pl->flops_alg;
  return TSG_OK;
}

int tsg_plan_describe(const tsg_plan* pl, char* buf, int len) {
  if (!pl) return -1;
  char tmp[160];
  if (pl->decoupled)
    std::snprintf(tmp, sizeof(tmp), "decoupled f=%d kappa=%.3g", pl->dec_f, pl->dec_kappa);
  else if (pl->use16)
    std::snprintf(tmp, sizeof(tmp), "lap16");
  else
    std::snprintf(tmp, sizeof(tmp), "%s", pl->fast == 3 ? "lap3" : pl->fast == 5 ? "lapd" : pl->fast == 6 ? "gsyd"
                                             : pl->fast == 1 ? "lap" : "generic");
  const int n = static_cast<int>(std::strlen(tmp));
  if (buf && len > 0) {
    std::strncpy(buf, tmp, static_cast<size_t>(len - 1));
    buf[len - 1] = 0;
  }
  return n;
}

// Status word of the solves enqueued since the last read (sticky: the
// kernels atomicMin into it, a gate timeout is negative so it wins), then
// re-armed to kNoStatus (memset 0x7f) in stream order.  Synchronises st.
static cudaError_t read_status(tsg_plan* pl, cudaStream_t st, int* hstat) {
  cudaError_t e = cudaMemcpyAsync(hstat, pl->counter, 2 * sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(pl->counter + 1, 0x7f, sizeof(int), st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e;
}

int tsg_plan_enqueue(tsg_plan* pl, const double* B, double* X) {
  if (!pl || !B || !X) return TSG_EINVAL;
  tsg_ctx* ctx = pl->ctx;
  TSG_CU(cudaSetDevice(ctx->device));
  return enqueue(pl, B, X, pl->ctx->stream, false);
}

int tsg_plan_transform(tsg_plan* pl, int dir, const double* in, double* out, void* stream) {
  if (!pl || !in || !out || in == out || pl->reduced_only) return TSG_EINVAL;
  tsg_ctx* ctx = pl->ctx;
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  TSG_CU(pl->w2.ensure(pl->N));
  // the slab-chain flags between the first two GEMMs are per call
  if (pl->flags) TSG_CU(tsg::reset_state(pl->flags, pl->ntiles, pl->counter, pl->aux, pl->aux_n, st));
  TSG_CU(transform_all(pl, in, out, pl->w2.p, dir == 0, st));
  return TSG_OK;
}

int tsg_plan_free_mode(const tsg_plan* pl) { return pl && pl->decoupled ? pl->dec_f : -1; }

int tsg_plan_set_serial(tsg_plan* pl, int serial) {
  if (!pl) return TSG_EINVAL;
  pl->knobs.serial = serial != 0;
  return TSG_OK;
}

int tsg_plan_sync(tsg_plan* pl, tsg_report* rep) {
  if (!pl) return TSG_EINVAL;
  tsg_ctx* ctx = pl->ctx;
  TSG_CU(cudaSetDevice(ctx->device));
  int hstat[2] = {0, kNoStatus};
  TSG_CU(read_status(pl, pl->ctx->stream, hstat));
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->flops_alg = pl->flops_alg;
    rep->flops_exec = pl->flops_exec;
    rep->zero_pivot_index = hstat[1] == kNoStatus || hstat[1] < 0 ? -1 : hstat[1];
    rep->kernel_launches = pl->launches;
  }
  // singular cells are reported through rep (the enqueue contract); a gate
  // timeout means some solve ran on incomplete inputs
  if (hstat[1] == tsg::kGateTimeout)
    return fail(ctx, TSG_ECUDA, "reduced solve: forward gate timed out (serialised launches)");
  return TSG_OK;
}

int tsg_plan_execute(tsg_plan* pl, const double* B, double* X, int inputs_on_device,
                     tsg_report* rep) {
  if (!pl) return TSG_EINVAL;
  tsg_ctx* ctx = pl->ctx;
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t bytes = static_cast<size_t>(pl->N) * sizeof(double);
  const double* din = B;
  double* dout = X;
  if (!inputs_on_device) {
    TSG_CU(pl->xdev.ensure(pl->N));
    din = pl->xdev.p;
    dout = pl->xdev.p;
  }
  cudaEvent_t* ev = ctx->ev;
  TSG_CU(cudaEventRecord(ev[0], st));
  if (!inputs_on_device)
    TSG_CU(cudaMemcpyAsync(pl->xdev.p, B, bytes, cudaMemcpyHostToDevice, st));
  TSG_CU(cudaEventRecord(ev[1], st));
  int rc = enqueue(pl, din, dout, st, true);
  if (rc != TSG_OK) return rc;
  TSG_CU(cudaEventRecord(ev[5], st));
  if (!inputs_on_device) TSG_CU(cudaMemcpyAsync(X, pl->xdev.p, bytes, cudaMemcpyDeviceToHost, st));
  TSG_CU(cudaEventRecord(ev[6], st));
  int hstat[2] = {0, kNoStatus};
  TSG_CU(read_status(pl, st, hstat));
  if (rep) {
    float t = 0;
    std::memset(rep, 0, sizeof(*rep));
    cudaEventElapsedTime(&t, ev[0], ev[1]);
    rep->t_h2d_ms = t;
    cudaEventElapsedTime(&t, ev[1], ev[2]);
    rep->t_fwd_ms = t;
    cudaEventElapsedTime(&t, ev[2], ev[3]);
    rep->t_solve_ms = t;
    cudaEventElapsedTime(&t, ev[3], ev[4]);
    rep->t_back_ms = t;
    cudaEventElapsedTime(&t, ev[5], ev[6]);
    rep->t_d2h_ms = t;
    cudaEventElapsedTime(&t, ev[0], ev[6]);
    rep->t_total_ms = t;
    rep->flops_alg = pl->flops_alg;
    rep->flops_exec = pl->flops_exec;
    rep->zero_pivot_index = hstat[1] == kNoStatus || hstat[1] < 0 ? -1 : hstat[1];
    rep->kernel_launches = pl->launches;
  }
  if (hstat[1] == tsg::kGateTimeout)
    return fail(ctx, TSG_ECUDA, "reduced solve: forward gate timed out (serialised launches)");
  if (hstat[1] != kNoStatus)
    return fail(ctx, TSG_ESINGULAR,
                "reduced solve: numerically singular base cell in tile " + std::to_string(hstat[1]));
  return TSG_OK;
}

int tsg_plan_execute_stream(tsg_plan* pl, int nrhs, const double* const* B, double* const* X,
                            tsg_report* rep) {
  if (!pl || nrhs < 0 || (nrhs > 0 && (!B || !X))) return TSG_EINVAL;
  tsg_ctx* ctx = pl->ctx;
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t bytes = static_cast<size_t>(pl->N) * sizeof(double);
  for (int s = 0; s < 2; ++s) {
    TSG_CU(pl->sin[s].ensure(pl->N));
    TSG_CU(pl->sout[s].ensure(pl->N));
  }
  // copy streams and events, released on every return path; an early error
  // return first drains the copy streams (they may still read the caller's
  // host buffers)
  struct Staging {
    cudaStream_t cin = nullptr, cout = nullptr;
    cudaEvent_t in_ready[2] = {}, solved[2] = {}, out_free[2] = {}, t0 = nullptr, t1 = nullptr;
    ~Staging() {
      if (cin) cudaStreamSynchronize(cin);
      if (cout) cudaStreamSynchronize(cout);
      for (cudaEvent_t e : {in_ready[0], in_ready[1], solved[0], solved[1], out_free[0], out_free[1], t0, t1})
        if (e) cudaEventDestroy(e);
      if (cin) cudaStreamDestroy(cin);
      if (cout) cudaStreamDestroy(cout);
    }
  } g;
  TSG_CU(cudaStreamCreateWithFlags(&g.cin, cudaStreamNonBlocking));
  TSG_CU(cudaStreamCreateWithFlags(&g.cout, cudaStreamNonBlocking));
  for (int s = 0; s < 2; ++s) {
    TSG_CU(cudaEventCreateWithFlags(&g.in_ready[s], cudaEventDisableTiming));
    TSG_CU(cudaEventCreateWithFlags(&g.solved[s], cudaEventDisableTiming));
    TSG_CU(cudaEventCreateWithFlags(&g.out_free[s], cudaEventDisableTiming));
  }
  TSG_CU(cudaEventCreate(&g.t0));
  TSG_CU(cudaEventCreate(&g.t1));
  cudaStream_t cin = g.cin, cout = g.cout;
  TSG_CU(cudaEventRecord(g.t0, st));
  TSG_CU(cudaStreamWaitEvent(cin, g.t0, 0));
  // status word of every solve, re-armed after each (singular cells,
  // gate timeouts), checked at the end
  DevBuf stat;
  TSG_CU(stat.ensure((static_cast<size_t>(std::max(nrhs, 1)) + 1) / 2));
  int* dstat = reinterpret_cast<int*>(stat.p);
  for (int i = 0; i < nrhs; ++i) {
    const int s = i & 1;
    // slot s input is free once solve i-2 finished
    if (i >= 2) TSG_CU(cudaStreamWaitEvent(cin, g.solved[s], 0));
    TSG_CU(cudaMemcpyAsync(pl->sin[s].p, B[i], bytes, cudaMemcpyHostToDevice, cin));
    TSG_CU(cudaEventRecord(g.in_ready[s], cin));
    TSG_CU(cudaStreamWaitEvent(st, g.in_ready[s], 0));
    if (i >= 2) TSG_CU(cudaStreamWaitEvent(st, g.out_free[s], 0));  // D2H of i-2 drained sout[s]
    const int rc = enqueue(pl, pl->sin[s].p, pl->sout[s].p, st, false);
    if (rc != TSG_OK) return rc;
    TSG_CU(cudaMemcpyAsync(dstat + i, pl->counter + 1, sizeof(int), cudaMemcpyDeviceToDevice, st));
    TSG_CU(cudaMemsetAsync(pl->counter + 1, 0x7f, sizeof(int), st));
    TSG_CU(cudaEventRecord(g.solved[s], st));
    TSG_CU(cudaStreamWaitEvent(cout, g.solved[s], 0));
    TSG_CU(cudaMemcpyAsync(X[i], pl->sout[s].p, bytes, cudaMemcpyDeviceToHost, cout));
    TSG_CU(cudaEventRecord(g.out_free[s], cout));
  }
  TSG_CU(cudaEventRecord(g.t1, cout));
  std::vector<int> hs(static_cast<size_t>(nrhs));
  if (nrhs > 0) TSG_CU(cudaMemcpyAsync(hs.data(), dstat, nrhs * sizeof(int), cudaMemcpyDeviceToHost, st));
  TSG_CU(cudaStreamSynchronize(cout));
  TSG_CU(cudaStreamSynchronize(st));
  int hstat[2] = {0, kNoStatus};
  for (int v : hs)
    if (v == tsg::kGateTimeout || (v != kNoStatus && hstat[1] == kNoStatus)) hstat[1] = v;
  if (rep) {
    float t = 0;
    std::memset(rep, 0, sizeof(*rep));
    cudaEventElapsedTime(&t, g.t0, g.t1);
    rep->t_total_ms = t;
    rep->flops_alg = pl->flops_alg * nrhs;
    rep->flops_exec = pl->flops_exec * nrhs;
    rep->zero_pivot_index = hstat[1] == kNoStatus || hstat[1] < 0 ? -1 : hstat[1];
    rep->kernel_launches = pl->launches * nrhs;
  }
  if (hstat[1] == tsg::kGateTimeout)
    return fail(ctx, TSG_ECUDA, "reduced solve: forward gate timed out (serialised launches)");
  if (hstat[1] != kNoStatus)
    return fail(ctx, TSG_ESINGULAR, "reduced solve: numerically singular base cell in tile " + std::to_string(hstat[1]));
  return TSG_OK;
}

int tsg_mode_multiply(tsg_ctx* ctx, int d, const int* dims, const double* X, int r, const double* A,
                      int mode, double* Y, const tsg_opts* opts) {
  if (!ctx) return TSG_EINVAL;
  if (d < 1 || d > TSG_MAX_ORDER || mode < 0 || mode >= d)
    return fail(ctx, TSG_EDIM, "mode_multiply: mode out of range");
  if (r <= 0) return fail(ctx, TSG_EDIM, "mode_multiply: A must have positive row count");
  int64_t N = 1, NY = 1;
  for (int m = 0; m < d; ++m) {
    if (dims[m] <= 0) return fail(ctx, TSG_EDIM, "dimensions must be positive");
    N *= dims[m];
    NY *= (m == mode ? r : dims[m]);
  }
  const bool on_dev = opts && opts->inputs_on_device;
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int n = dims[mode];
  DevBuf dx, dy, da, dat;
  const std::vector<double> at_h = [&] {
    std::vector<double> t(static_cast<size_t>(n) * r);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < r; ++i) t[j + static_cast<size_t>(i) * n] = A[i + static_cast<size_t>(j) * r];
    return t;
  }();
  TSG_CU(upload_mat(da, A, static_cast<size_t>(r) * n));
  TSG_CU(upload_mat(dat, at_h.data(), at_h.size()));
  const double* xin = X;
  double* yout = Y;
  if (!on_dev) {
    TSG_CU(upload_mat(dx, X, N));
    TSG_CU(dy.ensure(NY));
    xin = dx.p;
    yout = dy.p;
  }
  TSG_CU(tsg::mode_product(xin, yout, d, dims, mode, da.p, dat.p, r, 1.0, 0.0, st));
  if (!on_dev)
    TSG_CU(cudaMemcpyAsync(Y, dy.p, NY * sizeof(double), cudaMemcpyDeviceToHost, st));
  TSG_CU(cudaStreamSynchronize(st));
  return TSG_OK;
}

int tsg_residual(tsg_ctx* ctx, int family, int d, const int* dims, const double* const* A,
                 const double* Cm, const double* B, const double* X, int inputs_on_device,
                 double* out) {
  if (!ctx || !out) return TSG_EINVAL;
  if (d < 1 || d > TSG_MAX_ORDER) return fail(ctx, TSG_EDIM, "residual: order out of range");
  if (family == 1 && !Cm) return fail(ctx, TSG_EDIM, "residual: gsylv needs C");
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  int64_t N = 1;
  for (int m = 0; m < d; ++m) N *= dims[m];
  DevBuf db, dx, r, t1, t2, acc;
  std::vector<DevBuf> da(d), dat(d);
  double scale = 0, prod = 1;
  for (int m = 0; m < d; ++m) {
    const size_t nn = static_cast<size_t>(dims[m]) * dims[m];
    TSG_CU(upload_mat(da[m], A[m], nn));
    const std::vector<double> at = transpose(A[m], dims[m]);
    TSG_CU(upload_mat(dat[m], at.data(), nn));
    const double f = fro(A[m], nn);
    if (family == 0) scale += f;
    else if (m == 0) scale += f;
    else prod *= f;
  }
  DevBuf dc;
  if (family == 1) {
    const size_t nn = static_cast<size_t>(dims[0]) * dims[0];
    TSG_CU(upload_mat(dc, Cm, nn));
    scale += fro(Cm, nn) * prod;
  }
  const double* b = B;
  const double* x = X;
  if (!inputs_on_device) {
    TSG_CU(upload_mat(db, B, N));
    TSG_CU(upload_mat(dx, X, N));
    b = db.p;
    x = dx.p;
  }
  TSG_CU(r.ensure(N));
  TSG_CU(acc.ensure(3));
  TSG_CU(cudaMemcpyAsync(r.p, b, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (family == 0) {
    // r = B - sum_m X x_m A_m   (beta = 1 accumulation, disjoint slabs)
    for (int m = 0; m < d; ++m)
      TSG_CU(tsg::mode_product(x, r.p, d, dims, m, da[m].p, dat[m].p, dims[m], -1.0, 1.0, st));
  } else {
    TSG_CU(tsg::mode_product(x, r.p, d, dims, 0, da[0].p, dat[0].p, dims[0], -1.0, 1.0, st));
    TSG_CU(t1.ensure(N));
    TSG_CU(t2.ensure(N));
    TSG_CU(tsg::mode_product(x, t1.p, d, dims, 0, dc.p, nullptr, dims[0], 1.0, 0.0, st));
    double* cur = t1.p;
    double* oth = t2.p;
    for (int m = 1; m < d; ++m) {
      TSG_CU(tsg::mode_product(cur, oth, d, dims, m, da[m].p, dat[m].p, dims[m], 1.0, 0.0, st));
      std::swap(cur, oth);
    }
    TSG_CU(tsg::axpy(r.p, cur, -1.0, N, st));
  }
  TSG_CU(cudaMemsetAsync(acc.p, 0, 3 * sizeof(double), st));
  TSG_CU(tsg::sumsq(r.p, N, acc.p, st));
  TSG_CU(tsg::sumsq(x, N, acc.p + 1, st));
  TSG_CU(tsg::sumsq(b, N, acc.p + 2, st));
  double h[3];
  TSG_CU(cudaMemcpyAsync(h, acc.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  TSG_CU(cudaStreamSynchronize(st));
  const double num = std::sqrt(h[0]), den = scale * std::sqrt(h[1]) + std::sqrt(h[2]);
  *out = den == 0 ? (num == 0 ? 0.0 : std::numeric_limits<double>::infinity()) : num / den;
  return TSG_OK;
}

static int one_shot(tsg_ctx* ctx, int family, int d, const int* dims, const double* const* T,
                    const double* const* U, const double* Tc, const double* Z, int reduced,
                    const double* B, double* X, const tsg_opts* opts, tsg_report* rep) {
  tsg_plan* pl = nullptr;
  int rc = tsg_plan_create(ctx, family, d, dims, T, U, Tc, Z, reduced, opts, &pl);
  if (rc != TSG_OK) return rc;
  rc = tsg_plan_execute(pl, B, X, opts ? opts->inputs_on_device : 0, rep);
  tsg_plan_destroy(pl);
  return rc;
}

int tsg_laplace_solve(tsg_ctx* ctx, int d, const int* dims, const double* const* T,
                      const double* const* U, const double* B, double* X, const tsg_opts* opts,
                      tsg_report* rep) {
  return one_shot(ctx, 0, d, dims, T, U, nullptr, nullptr, 0, B, X, opts, rep);
}

int tsg_laplace_reduced(tsg_ctx* ctx, int d, const int* dims, const double* const* T,
                        const double* Bt, double* Xt, const tsg_opts* opts, tsg_report* rep) {
  return one_shot(ctx, 0, d, dims, T, nullptr, nullptr, nullptr, 1, Bt, Xt, opts, rep);
}

int tsg_gsylv_solve(tsg_ctx* ctx, int d, const int* dims, const double* S, const double* Tc,
                    const double* Q, const double* Z, const double* const* Ttail,
                    const double* const* Utail, const double* B, double* X, const tsg_opts* opts,
                    tsg_report* rep) {
  if (d < 2 || d > TSG_MAX_ORDER) return fail(ctx, TSG_EDIM, "order d out of range");
  const double* T[TSG_MAX_ORDER];
  const double* U[TSG_MAX_ORDER];
  T[0] = S;
  U[0] = Q;
  for (int m = 1; m < d; ++m) {
    T[m] = Ttail[m - 1];
    U[m] = Utail[m - 1];
  }
  return one_shot(ctx, 1, d, dims, T, U, Tc, Z, 0, B, X, opts, rep);
}

int tsg_gsylv_reduced(tsg_ctx* ctx, int d, const int* dims, const double* S, const double* Tc,
                      const double* const* Ttail, const double* Bt, double* Xt,
                      const tsg_opts* opts, tsg_report* rep) {
  if (d < 2 || d > TSG_MAX_ORDER) return fail(ctx, TSG_EDIM, "order d out of range");
  const double* T[TSG_MAX_ORDER];
  T[0] = S;
  for (int m = 1; m < d; ++m) T[m] = Ttail[m - 1];
  return one_shot(ctx, 1, d, dims, T, nullptr, Tc, nullptr, 1, Bt, Xt, opts, rep);
}

}  // extern "C"

namespace tsg_impl {

void fill_solve_args(const tsg_plan* pl, double* work, tsg::SolveArgs& a) {
  const int d = pl->d;
  a.family = pl->family;
  a.d = d;
  for (int m = 0; m < d; ++m) {
    a.dims[m] = pl->dims[m];
    a.stride[m] = pl->stride[m];
    a.T[m] = pl->T[m].p;
    a.tmode[m] = pl->tmode[m];
    a.eig[m] = pl->eig[m].p;
    a.pdat[m] = pl->pdat[m].p;
    a.dhat[m] = pl->dhat[m].p;
    a.vhat[m] = pl->vhat[m].p;
    a.ntiles_mode[m] = pl->ntiles_mode[m];
    a.bnd[m] = pl->bnd[m];
    a.rowtile[m] = pl->rowtile[m];
    if (pl->family == 1 && m >= 1) a.W[m] = pl->wchain[m].p;
  }
  a.Tc = pl->family == 1 ? pl->Tc.p : nullptr;
  a.X = work;
  a.ntiles = pl->ntiles;
  a.order = pl->order;
  a.ocoord = pl->ocoord;
  a.tiny = pl->tiny;
  a.refine = pl->refine;
  for (size_t m = 0; m < pl->tlog.size(); ++m) {
    a.tlog[m] = pl->tlog[m];
    a.tsh[m] = pl->tsh[m];
  }
  // one slab: the whole tensor
  a.nslab = 1;
  a.sys = 0;
  a.slo[0] = 0;
  a.slo[1] = pl->dims[d - 1];
  a.xs[0] = work;
}

cudaError_t launch_plan_solve(tsg_plan* pl, const tsg::SolveArgs& a, cudaStream_t st) {
  if (pl->use16) return tsg::launch_solve_lap16(a, st, &pl->solve_info);
  if (pl->fast == 5) return tsg::launch_solve_lapd(a, st, &pl->solve_info);
  if (pl->fast == 6) return tsg::launch_solve_gsyd(a, st, &pl->solve_info);
  if (pl->fast == 3) return tsg::launch_solve_lap3(pl->lt3, a, st, &pl->solve_info);
  if (pl->fast) return tsg::launch_solve_lap(a, st, &pl->solve_info);
  return tsg::launch_solve(a, st, &pl->solve_info);
}

}  // namespace tsg_impl

// All-mode transform in -> target (ping-pong through `other`): per-mode DMMA
// GEMMs, except consecutive small modes (n in {16, 24, 32, 40}), which go
// through the fused shared-memory pass two at a time (modes_small.cu).
cudaError_t transform_all(tsg_plan* pl, const double* in, double* target, double* other, bool fwd,
                          cudaStream_t st, const tsg::GemmArgs* gate0, cudaEvent_t after0, int i_lo, int i_hi,
                          const tsg::GemmArgs* last) {
  const int d = pl->d;
  struct Pass {
    int m;
    int kind;  // 0 GEMM, 1 small single, 2 small pair
  };
  std::vector<Pass> ps;
  static const bool small_on = [] {
    const char* e = std::getenv("TSG_SMALLMODES");
    return !e || std::atoi(e) != 0;
  }();
  auto skip = [&](int m) { return (pl->skip_mask >> m) & 1; };
  for (int m = 0; m < d;) {
    const int* dm = pl->dims.data();
    if (skip(m)) {
      ++m;
      continue;
    }
    if (small_on && m + 1 < d && !skip(m + 1) && tsg::small_pass_ok(d, dm, m, true)) {
      ps.push_back({m, 2});
      m += 2;
    } else {
      ps.push_back({m, small_on && tsg::small_pass_ok(d, dm, m, false) ? 1 : 0});
      m += 1;
    }
  }
  const int k = static_cast<int>(ps.size());
  if (k == 0) {  // every transform is the identity
    if (in != target)
      return cudaMemcpyAsync(target, in, pl->N * sizeof(double), cudaMemcpyDeviceToDevice, st);
    return cudaSuccess;
  }
  // slab chain: mode-1 CTAs start on the slabs the mode-0 GEMM has finished
  // (TSG_SCHAIN=0 at plan creation turns it off)
  const bool schain = pl->sdone[0] && k >= 2 && ps[0].m == 0 && ps[0].kind == 0 && ps[1].m == 1 &&
                      ps[1].kind == 0 && !pl->knobs.schain_off;
  int* sdone = pl->sdone[fwd ? 0 : 1];
  if (i_hi < 0 || i_hi > k) i_hi = k;
  // pass i reads the previous pass's output (ping-pong ending in target)
  const double* src = i_lo == 0 ? in : (((k - i_lo) % 2 == 0) ? target : other);
  for (int i = i_lo; i < i_hi; ++i) {
    double* dst = ((k - 1 - i) % 2 == 0) ? target : other;
    const int m = ps[i].m;
    const double* A = fwd ? pl->Fwd[m].p : pl->Bwd[m].p;
    const double* At = fwd ? pl->FwdT[m].p : pl->BwdT[m].p;
    cudaError_t e;
    if (ps[i].kind == 0) {
      // GEMM after GEMM: programmatic launch (the next pass's CTAs are
      // scheduled while this one drains; pdl_wait() orders the data).
      tsg::GemmArgs chain{};
      if (i == 0 && gate0) chain = *gate0;
      chain.pdl = (i == 0 && gate0) || (i > 0 && ps[i - 1].kind == 0) ? 1 : 0;
      if (schain && i == 0) {
        chain.dflags = sdone;
        chain.depoch = 1;
      } else if (schain && i == 1) {
        chain.pflags = sdone;
        chain.pepoch = 1;
        chain.ptm = pl->s_tm;
        chain.pbn = pl->s_bn;
        chain.pcpb = pl->dims[1];
        chain.pdesc = gate0 && gate0->wflags ? 1 : 0;  // gated mode 0 runs last columns first
      }
      if (last && i == k - 1) {  // the last forward GEMM feeding the trailing cube
        chain.pdl = last->pdl;
        chain.nowait = last->nowait;
        chain.dflags = last->dflags;
        chain.depoch = last->depoch;
        chain.drev = last->drev;
      }
      const tsg::GemmArgs* opt = &chain;
      e = tsg::mode_product(src, dst, d, pl->dims.data(), m, A, At, pl->dims[m], 1.0, 0.0, st,
                            nullptr, opt);
    } else {
      const double* B = ps[i].kind == 2 ? (fwd ? pl->Fwd[m + 1].p : pl->Bwd[m + 1].p) : nullptr;
      e = tsg::mode_pair_small(src, dst, d, pl->dims.data(), m, ps[i].kind == 2, A, B, st);
    }
    if (e != cudaSuccess) return e;
    ++pl->launches;
    if (i == (schain ? 1 : 0) && after0) {
      e = cudaEventRecord(after0, st);
      if (e != cudaSuccess) return e;
    }
    src = dst;
  }
  return cudaSuccess;
}

namespace {

// Enqueue the whole pipeline on `st` (fwd transforms, solve, back transforms).
int enqueue(tsg_plan* pl, const double* in, double* out, cudaStream_t st, bool timing) {
  tsg_ctx* ctx = pl->ctx;
  const int d = pl->d;
  cudaEvent_t* ev = ctx->ev;
  pl->launches = 0;
  double* work = nullptr;
  // Solve state reset first, so the forward GEMMs and the solve follow each
  // other directly (programmatic launches).
  TSG_CU(tsg::reset_state(pl->flags, pl->ntiles, pl->counter, pl->aux, pl->aux_n, st));
  if (pl->decoupled) {
    TSG_CU(transform_all(pl, in, pl->w1.p, pl->w2.p, true, st));
    if (timing) TSG_CU(cudaEventRecord(ev[2], st));
    tsg::FibreArgs fa = pl->fib;
    fa.X = pl->w1.p;
    fa.counter = pl->counter;
    fa.status = pl->counter + 1;
    static unsigned long long* fprof = nullptr;
    if (pl->knobs.prof) {
      if (!fprof) TSG_CU(cudaMalloc(&fprof, 16 * sizeof(unsigned long long)));
      TSG_CU(cudaMemsetAsync(fprof, 0, 16 * sizeof(unsigned long long), st));
      fa.prof = fprof;
    }
    TSG_CU(tsg::launch_fibre_solve(fa, ctx->device, st, &pl->solve_info));
    ++pl->launches;
    if (pl->knobs.prof) {
      unsigned long long h[16];
      TSG_CU(cudaMemcpyAsync(h, fprof, sizeof(h), cudaMemcpyDeviceToHost, st));
      TSG_CU(cudaStreamSynchronize(st));
      const double nbw = h[6] ? static_cast<double>(h[6]) : 1.0;
      std::fprintf(stderr, "[tsg profw] per block per warp (cycles): load %.0f  butterfly+pack %.0f  barrier-A waits %.0f  leader subst %.0f  helper partials %.0f  store %.0f  (blocks x warps %.0f)\n",
                   h[0] / nbw, h[1] / nbw, h[2] / nbw, h[3] / nbw, h[4] / nbw, h[5] / nbw, nbw);
      std::fprintf(stderr, "[tsg profw] leaders per sub-partition %llu %llu %llu %llu, helpers %llu %llu %llu %llu\n",
                   h[8], h[9], h[10], h[11], h[12], h[13], h[14], h[15]);
    }
    if (timing) TSG_CU(cudaEventRecord(ev[3], st));
    TSG_CU(transform_all(pl, pl->w1.p, out, pl->w2.p, false, st));
    if (timing) TSG_CU(cudaEventRecord(ev[4], st));
    return TSG_OK;
  }
  const bool want_trace = pl->knobs.trace;
  const bool want_prof = pl->knobs.prof;
  // serial plans run every kernel after its predecessor: the back transform
  // after the solve, no trailing cube (bench kernel timing).
  const bool gate_off = pl->knobs.serial;
  // The cube grid waits on the NEXT kernel (the last forward GEMM): only
  // with concurrent kernels.  Serialising tools (Nsight Compute / Systems,
  // compute-sanitizer, CUDA_LAUNCH_BLOCKING=1) run without it.
  static const bool serialized = [] {
    const char* lb = std::getenv("CUDA_LAUNCH_BLOCKING");
    return (lb && std::atoi(lb) != 0) || std::getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") ||
           std::getenv("NV_TPS_LAUNCH_TOKEN") || std::getenv("CUDA_INJECTION64_PATH");
  }();
  const bool cubed = pl->cube > 0 && !want_trace && !want_prof && !gate_off && !serialized;
  // Forward transforms: outputs alternate w2/w1 and end in w1.
  if (!pl->reduced_only && cubed) {
    // all passes but the last; then the cube grid (resident on a few SMs,
    // waiting per tile on the last GEMM's done flags); then the last GEMM
    // as its programmatic dependent (inputs complete: no griddepcontrol.wait)
    TSG_CU(transform_all(pl, in, pl->w1.p, pl->w2.p, true, st, nullptr, nullptr, 0, 2));
    if (timing) TSG_CU(cudaEventRecord(ev[2], st));
    work = pl->w1.p;
    tsg::SolveArgs c{};
    tsg_impl::fill_solve_args(pl, work, c);
    c.flags = pl->flags;
    c.fs[0] = pl->flags;
    c.counter = pl->fdone + pl->fdone_n;
    c.status = pl->counter + 1;
    c.epoch = 1;
    c.order = pl->order1;
    c.ocoord = pl->ocoord1;
    c.ntiles = pl->ntiles1;
    c.gflags = pl->fdone;
    c.gepoch = 1;
    c.gbm = pl->fg_bm;
    c.gbn = pl->fg_bn;
    c.gtm = pl->fg_tm;
    c.max_grid = pl->cube_grid;
    c.dbg = pl->knobs.dbg;
    TSG_CU(tsg::launch_solve_lap16(c, st, nullptr));
    ++pl->launches;
    tsg::GemmArgs lastg{};
    lastg.pdl = 1;
    lastg.nowait = 1;
    lastg.dflags = pl->fdone;
    lastg.depoch = 1;
    lastg.drev = 1;
    TSG_CU(transform_all(pl, in, pl->w1.p, pl->w2.p, true, st, nullptr, nullptr, 2, 3, &lastg));
  } else if (!pl->reduced_only) {
    TSG_CU(transform_all(pl, in, pl->w1.p, pl->w2.p, true, st));
    work = pl->w1.p;
  } else {
    work = out;
    if (in != out)
      TSG_CU(cudaMemcpyAsync(out, in, pl->N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  if (timing && !cubed) TSG_CU(cudaEventRecord(ev[2], st));
  // Reduced solve.
  tsg::SolveArgs a{};
  tsg_impl::fill_solve_args(pl, work, a);
  a.flags = pl->flags;
  a.fs[0] = pl->flags;
  a.counter = pl->counter;
  a.status = pl->counter + 1;
  a.epoch = 1;
  if (cubed) {  // the cube's tiles are the first grid's
    a.order = pl->order2;
    a.ocoord = pl->ocoord2;
    a.ntiles = pl->ntiles2;
    // programmatic dependent of the last forward GEMM: CTAs take the SMs its
    // last wave frees and start on the tiles whose right-hand side is done
    static const bool main_gate = [] {
      const char* e = std::getenv("TSG_CUBE_MAINGATE");
      return !e || std::atoi(e) != 0;
    }();
    if (main_gate) {
      a.gflags = pl->fdone;
      a.gepoch = 1;
      a.gbm = pl->fg_bm;
      a.gbn = pl->fg_bn;
      a.gtm = pl->fg_tm;
      a.gate_pdl = 1;
    }
  }
  a.tiny = pl->tiny;
  a.refine = pl->refine;
  a.dbg = pl->knobs.dbg;
  static unsigned long long* trace = nullptr;
  static int64_t trace_n = 0;
  if (want_trace) {
    if (trace_n < 4 * pl->ntiles) {
      if (trace) cudaFree(trace);
      cudaMalloc(&trace, 4 * pl->ntiles * sizeof(unsigned long long));
      trace_n = 4 * pl->ntiles;
    }
    cudaMemsetAsync(trace, 0, 4 * pl->ntiles * sizeof(unsigned long long), st);
    a.trace = trace;
    a.ntiles_total = pl->ntiles;
  }
  static unsigned long long* prof = nullptr;
  if (want_prof) {
    if (!prof) cudaMalloc(&prof, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(prof, 0, 16 * sizeof(unsigned long long), st);
    a.prof = prof;
  }
  TSG_CU(tsg_impl::launch_plan_solve(pl, a, st));
  ++pl->launches;
  if (want_trace) {
    // per hyperplane: count, first and last release (us from the first release)
    std::vector<unsigned long long> tr(pl->ntiles), tr4(4 * pl->ntiles);
    cudaMemcpyAsync(tr4.data(), trace, 4 * pl->ntiles * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    std::copy(tr4.begin(), tr4.begin() + pl->ntiles, tr.begin());
    unsigned long long t0 = ~0ull;
    for (auto v : tr) t0 = std::min(t0, v);
    std::vector<int> hp(pl->ntiles);
    int H = 0;
    for (int64_t t = 0; t < pl->ntiles; ++t) {
      int64_t r = t;
      int h = 0;
      for (int m = 0; m < d; ++m) {
        h += static_cast<int>(r % pl->ntiles_mode[m]);
        r /= pl->ntiles_mode[m];
      }
      hp[t] = h;
      H = std::max(H, h);
    }
    std::vector<double> lo(H + 1, 1e30), hi(H + 1, 0);
    std::vector<int> cnt(H + 1, 0);
    for (int64_t t = 0; t < pl->ntiles; ++t) {
      const double v = (tr[t] - t0) * 1e-3;
      lo[hp[t]] = std::min(lo[hp[t]], v);
      hi[hp[t]] = std::max(hi[hp[t]], v);
      cnt[hp[t]]++;
    }
    std::fprintf(stderr, "[tsg trace] hyperplane: tiles first_us last_us\n");
    for (int h = H; h >= 0; --h)
      std::fprintf(stderr, "[tsg trace] %3d %5d %9.1f %9.1f\n", h, cnt[h], lo[h], hi[h]);
    if (tr4[pl->ntiles] | tr4[pl->ntiles + 1]) {  // -DL16_TRACE2=1 build: per-tile phases
      std::vector<double> c2f(H + 1, 0), f2d(H + 1, 0), d2r(H + 1, 0), cl(H + 1, 0);
      for (int64_t t = 0; t < pl->ntiles; ++t) {
        const double rel = tr[t], cla = tr4[pl->ntiles + t], far = tr4[2 * pl->ntiles + t],
                     dn = tr4[3 * pl->ntiles + t];
        const double f = far > 0 ? far : cla;
        c2f[hp[t]] += (f - cla) * 1e-3;
        f2d[hp[t]] += (dn - f) * 1e-3;
        d2r[hp[t]] += (rel - dn) * 1e-3;
        cl[hp[t]] += (cla - t0) * 1e-3;
      }
      std::fprintf(stderr, "[tsg trace2] hp tiles claim_us claim->far_done far_done->chunks_done chunks_done->release (avg us)\n");
      for (int h = H; h >= 0; --h)
        std::fprintf(stderr, "[tsg trace2] %3d %5d %9.1f %9.1f %9.1f %9.1f\n", h, cnt[h], cl[h] / cnt[h],
                     c2f[h] / cnt[h], f2d[h] / cnt[h], d2r[h] / cnt[h]);
    }
  }
  if (want_prof) {
    unsigned long long h[16];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const double nt = h[8] ? static_cast<double>(h[8]) : 1.0;
    if (pl->fast == 5)
      std::fprintf(stderr, "[tsg profd] tiles=%.0f cycles/tile: claim+geom %.0f gather %.0f far %.0f near %.0f base %.0f scatter+rel %.0f\n",
                   nt, h[0] / nt, h[1] / nt, h[2] / nt, h[3] / nt, h[4] / nt, h[5] / nt);
    else if (pl->use16 && tsg::lap16_decoupled())
      std::fprintf(stderr, "[tsg prof16d] tiles=%.0f cycles/tile (consumer 0): wait tile info %.0f chunks (incl. ring waits) %.0f B~ box wait %.0f flush %.0f bases wait %.0f base case %.0f scatter+release %.0f\n",
                   nt, h[0] / nt, h[1] / nt, h[2] / nt, h[3] / nt, h[4] / nt, h[5] / nt, h[6] / nt);
    else if (pl->use16)
      std::fprintf(stderr, "[tsg prof16] tiles=%.0f cycles/tile (consumer 0): claim+geom %.0f first-box %.0f chunks %.0f flush %.0f diag %.0f scatter+rel %.0f | producer: flag waits %.0f ring waits+issue %.0f\n",
                   nt, h[0] / nt, h[1] / nt, h[2] / nt, h[3] / nt, h[4] / nt, h[5] / nt, h[6] / nt, h[7] / nt);
    else
    std::fprintf(stderr, "[tsg prof] tiles=%.0f cycles/tile: setup %.0f stage %.0f update(near) %.0f farwait|That+fwdT %.0f far|wave %.0f diag|backT %.0f scatter %.0f | idle/queue %.0f\n",
                 nt, h[0] / nt, h[1] / nt, h[2] / nt, h[3] / nt, h[4] / nt, h[5] / nt, h[6] / nt, h[7] / nt);
  }
  if (pl->knobs.verbose)
    std::fprintf(stderr, "[tsg] solve grid=%d block=%d smem=%d ctas/sm=%d tiles=%lld refine=%d cond=%.3g\n",
                 pl->solve_info.grid, pl->solve_info.block, pl->solve_info.smem_bytes,
                 pl->solve_info.ctas_per_sm, static_cast<long long>(pl->ntiles), pl->refine,
                 pl->max_cond);
  // Back transforms: outputs alternate (w2, out) and end in `out`.  With the
  // gate, the mode-0 pass follows the solve directly (programmatic launch),
  // so the solve/back split point moves after it.
  // Serial plans run the back transform after the solve, so the bench can
  // time the solve kernel alone.
  const bool gated = pl->gate_groups > 0 && !want_trace && !want_prof && !gate_off;
  if (timing && !gated) TSG_CU(cudaEventRecord(ev[3], st));
  if (!pl->reduced_only) {
    tsg::GemmArgs gate{};
    gate.wflags = pl->flags;
    gate.woff = pl->gate_off;
    gate.wids = pl->gate_ids;
    gate.wepoch = 1;
    gate.wgroups = pl->gate_groups;
    gate.pdl = 1;
    TSG_CU(transform_all(pl, work, out, pl->w2.p, false, st, gated ? &gate : nullptr,
                         gated && timing ? ev[3] : nullptr));
  }
  if (timing) TSG_CU(cudaEventRecord(ev[4], st));
  if (cubed && pl->knobs.dbg_fdone) {  // development: unreleased forward-gate tiles
    std::vector<int> fd(pl->fdone_n);
    cudaMemcpyAsync(fd.data(), pl->fdone, pl->fdone_n * sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    int nun = 0;
    for (int i = 0; i < pl->fdone_n; ++i)
      if (fd[i] != 1) {
        if (nun < 12) std::fprintf(stderr, "[tsg dbg] fdone[%d] (mt %d nt %d) = %d\n", i, i % pl->fg_tm, i / pl->fg_tm, fd[i]);
        ++nun;
      }
    std::fprintf(stderr, "[tsg dbg] fdone unreleased %d of %d (tm %d, bm %d, bn %d)\n", nun, pl->fdone_n, pl->fg_tm,
                 pl->fg_bm, pl->fg_bn);
  }
  return TSG_OK;
}

template <typename V>
cudaError_t upload_owned(tsg_plan* pl, const V& v, const typename V::value_type** out) {
  using E = typename V::value_type;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, std::max<size_t>(v.size(), 1) * sizeof(E));
  if (e != cudaSuccess) return e;
  pl->owned.push_back(p);
  e = cudaMemcpy(p, v.data(), v.size() * sizeof(E), cudaMemcpyHostToDevice);
  *out = static_cast<const E*>(p);
  return e;
}

// Eigen-decoupled path.  Laplace plans with transforms: every
// mode but one free mode f > 0 with a well-conditioned real block-eigenbasis
// (prod kappa_2 <= kDecoupleKappa); the fibres along f are solved with the
// Kronecker SUM of the other modes' eigenvalues as shift.  gsylv plans: the
// tail modes 1..d-1 in their eigenbases, f = 0: the pencil (S + z Tc) per
// fibre with z the PRODUCT of the tail eigenvalues (wide kernel only).  The
// chunk mode (whose cells form a block's units) is mode 0 for Laplace and
// mode 1 for gsylv.  TSG_DECOUPLE=0 turns it off, TSG_DECOUPLE_NFMAX bounds
// n_f (default 1024).
int try_decouple(tsg_plan* pl, const double* const* T, const double* const* U, const double* Tc) {
  tsg_ctx* ctx = pl->ctx;
  const int d = pl->d;
  const int* dims = pl->dims.data();
  const bool gs = pl->family == 1;
  const char* env = std::getenv("TSG_DECOUPLE");
  if (pl->reduced_only || tsg_impl::g_force_lap3 || (env && std::atoi(env) == 0)) return TSG_OK;
  if (pl->family > 1 || d < 2) return TSG_OK;
  const int cm = gs ? 1 : 0;  // chunk mode
  if (gs ? d - 2 > tsg::kFibreMaxS : d - 1 > tsg::kFibreMaxS) return TSG_OK;
  const char* ne = std::getenv("TSG_DECOUPLE_NFMAX");
  const int nfmax = ne ? std::atoi(ne) : 1024;
  std::vector<tsg_impl::ModeEigen> me(d);
  std::vector<int> ok(d, 0);
  for (int m = gs ? 1 : 0; m < d; ++m) ok[m] = tsg_impl::mode_eigen(T[m], dims[m], me[m]) ? 1 : 0;
  int best = -1;
  double best_prod = 0;
  if (gs) {
    double prod = 1;
    for (int m = 1; m < d; ++m) prod *= ok[m] ? me[m].kappa : 1e300;
    if (dims[0] <= nfmax && prod <= tsg_impl::kDecoupleKappa) {
      best = 0;
      best_prod = prod;
    }
  } else {
    for (int f = 1; f < d; ++f) {
      if (dims[f] > nfmax || (pl->force_f >= 0 && f != pl->force_f)) continue;
      double prod = 1;
      for (int m = 0; m < d; ++m)
        if (m != f) prod *= ok[m] ? me[m].kappa : 1e300;
      if (!(prod <= tsg_impl::kDecoupleKappa)) continue;
      const double kf = ok[f] ? me[f].kappa : 1e300;
      if (best < 0 || dims[f] < dims[best] || (dims[f] == dims[best] && kf > (ok[best] ? me[best].kappa : 1e300))) {
        best = f;
        best_prod = prod;
      }
    }
  }
  if (best < 0) return TSG_OK;
  const int f = best;
  const int nf = dims[f];
  // S' = the eigen modes other than the chunk mode
  std::vector<int> sp;
  for (int m = 0; m < d; ++m)
    if (m != f && m != cm) sp.push_back(m);
  int nsc = 0;
  for (int m : sp) {
    bool cx = false;
    for (const auto& c : me[m].cells) cx = cx || c.size == 2;
    nsc += cx ? 1 : 0;
  }
  if (!gs) {
    const std::vector<int8_t> code = block_codes(T[f], nf);
    for (int i = 0; i < nf; ++i)
      if (code[i] == 1) {
        const double p = at(T[f], nf, i, i), b = at(T[f], nf, i, i + 1), c = at(T[f], nf, i + 1, i),
                     q = at(T[f], nf, i + 1, i + 1);
        if (!(0.25 * (p - q) * (p - q) + b * c < 0)) return TSG_OK;  // not in standard form
      }
    const size_t tb = nf <= 64 ? static_cast<size_t>(nf) * nf * 8 : 0;
    if (100 * 1024 <= tb + ((static_cast<size_t>(nf) * 8 + 4) << nsc) * 2) return TSG_OK;
  }
  tsg::FibreArgs& a = pl->fib;
  a = tsg::FibreArgs{};
  a.nf = nf;
  a.sf = pl->stride[f];
  a.gs = gs ? 1 : 0;
  a.sc = pl->stride[cm];
  {
    std::vector<double> tt(static_cast<size_t>(nf) * nf), fc(4 * static_cast<size_t>(nf), 0.0);
    for (int i = 0; i < nf; ++i)
      for (int j = 0; j < nf; ++j) tt[static_cast<size_t>(i) * nf + j] = T[f][i + static_cast<size_t>(j) * nf];
    const std::vector<int8_t> code = block_codes(T[f], nf);
    for (int i = 0; i < nf; ++i) {
      fc[4 * i] = code[i];
      if (code[i] == 1 && !gs) {
        const double p = at(T[f], nf, i, i), b = at(T[f], nf, i, i + 1), c = at(T[f], nf, i + 1, i),
                     q = at(T[f], nf, i + 1, i + 1);
        const double disc = 0.25 * (p - q) * (p - q) + b * c;
        const double re = 0.5 * (p + q), w = disc < 0 ? std::sqrt(-disc) : 0.0;
        const double r2 = disc < 0 ? 0.0 : std::sqrt(disc);
        // eigenvalues re +- i w (complex pair) or re +- r2 (real pair: stored as w = i r2
        // is not representable; use the nearer-to-zero bound via re and r2 in the check)
        fc[4 * i + 1] = fc[4 * i + 5] = re;
        fc[4 * i + 2] = fc[4 * i + 6] = w;
        fc[4 * i + 3] = fc[4 * i + 7] = r2;
      }
    }
    TSG_CU(upload_owned(pl, tt, &a.Tt));
    TSG_CU(upload_owned(pl, fc, &a.fcell));
    if (gs) {
      std::vector<double> tc(static_cast<size_t>(nf) * nf);
      for (int i = 0; i < nf; ++i)
        for (int j = 0; j < nf; ++j) tc[static_cast<size_t>(i) * nf + j] = Tc[i + static_cast<size_t>(j) * nf];
      TSG_CU(upload_owned(pl, tc, &a.Tct));
    }
  }
  int64_t nblk_rest = 1;
  for (int m : sp) {
    const int s = a.ns++;
    a.sstride[s] = pl->stride[m];
    a.ncell[s] = static_cast<int>(me[m].cells.size());
    TSG_CU(upload_owned(pl, me[m].cells, &a.cells[s]));
    nblk_rest *= a.ncell[s];
  }
  // chunks of whole chunk-mode cells within the shared-memory budget: the
  // register kernel for n_f <= 24 (three CTAs per SM), else the team DMMA
  // kernel (blocks of <= kWideCols real columns; fewer when a long free mode
  // would not leave room for two CTAs per SM), else the DMMA-blocked kernel
  // (TSG_FIBRE_WIDE=0; Laplace only)
  const bool small = nf <= 24 && !gs;
  int W = 0;
  int ncell_s = 0;
  for (int m : sp) ncell_s += static_cast<int>(me[m].cells.size());
  const int cell_smem = ncell_s <= 1024 ? ncell_s : 0;
  bool wide = false;
  if (small) {
    // two block buffers (the next block streams in while one is solved) in
    // ~100 KB: two CTAs per SM, blocks of >= 128 complex jobs for C3 (C3
    // fibre solve 5.7 ms at 72 KB / 3 CTAs, 5.25 ms at 100 KB; TSG_FIBRE_SMEM_KB)
    const int NF = nf <= 8 ? 8 : nf <= 16 ? 16 : 24;
    const long avail = ((std::getenv("TSG_FIBRE_SMEM_KB") ? std::atoi(std::getenv("TSG_FIBRE_SMEM_KB")) : 100) * 1024 - 2 * 128 * 32 - cell_smem * 24) / 8 - NF * NF - 3 * NF;
    W = static_cast<int>(std::min<long>(avail / (2 * (static_cast<long>(nf) << nsc)), 128));
  } else {
    const char* we = std::getenv("TSG_FIBRE_WIDE");
    if (gs || !(we && std::atoi(we) == 0)) {
      for (int mc = tsg::kWideCols; mc >= 8 && !wide; mc /= 2) {
        if (tsg::fibre_wide_smem(nf, mc, cell_smem, 0, gs ? 1 : 0) > 110 * 1024) continue;
        W = mc >> nsc;
        wide = W >= 2;
      }
    }
    if (!wide) {
      if (gs) return TSG_OK;
      const size_t per_row = (static_cast<size_t>(nf) * 8 + 24) << nsc;
      const size_t fixed = static_cast<size_t>(nf) * 16 * 8 + 128 * 32 + 16 + cell_smem * 24;
      W = 108 * 1024 > fixed ? static_cast<int>(std::min<size_t>((108 * 1024 - fixed) / per_row, 128)) : 0;
    }
  }
  if (W < 2) return TSG_OK;  // not admissible: the tile kernels keep the plan
  const int ncm = dims[cm];
  std::vector<int> chunk{0}, cellrow0(ncm);
  const auto& c0 = me[cm].cells;
  for (int c = 0; c < static_cast<int>(c0.size()); ++c) {
    for (int r = c0[c].start; r < c0[c].start + c0[c].size; ++r) cellrow0[r] = c;
    if (c0[c].start + c0[c].size - chunk.back() > W) chunk.push_back(c0[c].start);
  }
  chunk.push_back(ncm);
  int wmax = 0;
  for (size_t q = 0; q + 1 < chunk.size(); ++q) wmax = std::max(wmax, chunk[q + 1] - chunk[q]);
  a.nchunk = static_cast<int>(chunk.size()) - 1;
  TSG_CU(upload_owned(pl, chunk, &a.chunk_lo));
  {
    std::vector<int> u0{0};
    std::vector<tsg::FibreUnit> units;
    for (int q = 0; q < a.nchunk; ++q) {
      int npb = 0;
      for (int c = cellrow0[chunk[q]]; c < static_cast<int>(c0.size()) && c0[c].start < chunk[q + 1]; ++c) {
        tsg::FibreUnit un{};
        un.rl0 = c0[c].start - chunk[q];
        un.pair0 = c0[c].size == 2 ? 1 : 0;
        un.npair_before = npb;
        un.sr = c0[c].re;
        un.si = un.pair0 ? -c0[c].im : 0.0;
        npb += un.pair0;
        units.push_back(un);
      }
      u0.push_back(static_cast<int>(units.size()));
    }
    TSG_CU(upload_owned(pl, u0, &a.chunk_u0));
    TSG_CU(upload_owned(pl, units, &a.units));
  }
  a.cell_smem = cell_smem;
  TSG_CU(upload_owned(pl, cellrow0, &a.cellrow0));
  TSG_CU(upload_owned(pl, c0, &a.cell0));
  a.maxcol = wmax << nsc;
  a.small = small && tsg::fibre_small_ok(nf, wmax) ? 1 : 0;
  if (const char* e = std::getenv("TSG_FIBRE_SMALL")) a.small = a.small && std::atoi(e) != 0;
  a.wide = !a.small && wide ? 1 : 0;
  a.big = a.small || a.wide ? 0 : 1;
  if (const char* e = std::getenv("TSG_FIBRE_BIG")) a.big = a.big && std::atoi(e) != 0;
  if (gs && !a.wide) return TSG_OK;
  if (a.big || a.wide) {
    // row blocks of f: <= 8 rows, never splitting a 2x2 cell
    const std::vector<int8_t> code = block_codes(T[f], nf);
    std::vector<int> rb{0};
    while (rb.back() < nf) {
      int e = std::min(rb.back() + 8, nf);
      if (e < nf && code[e] == 2) --e;
      rb.push_back(e);
    }
    a.nrb = static_cast<int>(rb.size()) - 1;
    TSG_CU(upload_owned(pl, rb, &a.rb));
    std::vector<unsigned> rbc(a.nrb, 0u);
    for (int q = 0; q < a.nrb; ++q)
      for (int i = rb[q]; i < rb[q + 1]; ++i) rbc[q] |= static_cast<unsigned>(code[i]) << (2 * (i - rb[q]));
    TSG_CU(upload_owned(pl, rbc, &a.rbcode));
    a.pitch = tsg::fibre_pitch(a.maxcol);
  }
  a.nblocks = static_cast<int64_t>(a.nchunk) * nblk_rest;
  if (a.nblocks >= (int64_t{1} << 31)) return TSG_OK;  // the kernels index blocks in 32 bits
  // folded transforms of the eigen modes (gsylv mode 0 keeps Q^T / Z)
  for (int m = 0; m < d; ++m) {
    if (m == f || ((pl->skip_mask >> m) & 1)) continue;
    const int n = dims[m];
    const size_t nn = static_cast<size_t>(n) * n;
    const std::vector<double> ut = transpose(U[m], n);
    const std::vector<double> fw = tsg_impl::matmul(me[m].Pinv.data(), ut.data(), n);
    const std::vector<double> bw = tsg_impl::matmul(U[m], me[m].P.data(), n);
    const std::vector<double> fwt = transpose(fw.data(), n), bwt = transpose(bw.data(), n);
    TSG_CU(upload_mat(pl->Fwd[m], fw.data(), nn));
    TSG_CU(upload_mat(pl->FwdT[m], fwt.data(), nn));
    TSG_CU(upload_mat(pl->Bwd[m], bw.data(), nn));
    TSG_CU(upload_mat(pl->BwdT[m], bwt.data(), nn));
  }
  a.tiny = pl->tiny;
  pl->decoupled = 1;
  pl->dec_f = f;
  pl->dec_kappa = best_prod;
  pl->tile_ext.assign(d, 2);
  pl->tile_ext[cm] = wmax;
  pl->tile_ext[f] = nf;
  pl->ntiles_mode.assign(d, 1);
  if (pl->knobs.verbose)
    std::fprintf(stderr, "[tsg] decoupled solve (%s): free mode %d (n=%d), prod kappa %.3g, blocks %lld, maxcol %d\n",
                 gs ? "gsylv" : "laplace", f, nf, best_prod, static_cast<long long>(a.nblocks), a.maxcol);
  return TSG_OK;
}


}  // namespace
