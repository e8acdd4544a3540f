// Complex-scalar solves on the GPU: the C-ABI entry
// points tsg_z* of include/tsylv_gpu.h behind solve_laplace<Complex>
// (laplace.hpp:324-344), solve_gsylv<Complex> (gsylv.hpp:311-331), their
// reduced forms (laplace_recursive / laplace_merged / gsylv_recursive /
// gsylv_merged and the d = 2 solvers for T = Complex), mode_multiply<Complex>
// (tensor.hpp:187-231) and oracle::residual<Complex> (oracle.hpp:233-268).
//
// Complex Schur factors are strictly upper triangular (zgees/zgges), so every
// mode has a plain eigenbasis T_m P_m = P_m diag(T_m), P_m unit upper
// triangular, computed here by back substitution.  Reduced solve:
//
//  * decoupled (default): all modes but one free mode f go into their
//    eigenbases; each fibre along f solves (T_f + sigma I) x = r (Laplace,
//    sigma = sum of the other modes' eigenvalues) or (S + z Tc) x = r
//    (gsylv, f = 0, z = product of the tail eigenvalues) — zfibre_kernel.
//    With prod_{m != f} kappa(P_m) <= kFoldKappa the eigenbasis change is
//    folded into the Schur transforms (one GEMM per mode and direction);
//    up to kRefineKappa the solve runs in the Schur basis with the eigenbasis
//    changes explicit and kRefineSteps steps of iterative refinement against
//    the triangular operator (rounding of the basis change is amplified by
//    kappa; refinement removes it).
//  * wavefront (Laplace, worse bases or defective T): the triangular
//    Kronecker sum solved hyperplane by hyperplane (zlevel_kernel) — exact
//    back substitution, no basis change.
//  gsylv bases beyond kRefineKappa refine with more steps.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/tsylv_gpu.h"
#include "plan_impl.h"
#include "util.h"
#include "zsolve.h"

namespace {

using C = std::complex<double>;
using tsg_impl::fail;

constexpr double kFoldKappa = 1e4;
constexpr double kRefineKappa = 1e12;
constexpr int kRefineSteps = 2;

const C* cptr(const double* p) { return reinterpret_cast<const C*>(p); }

struct ZMat {
  int n = 0;
  std::vector<C> a;  // column-major n x n
  C& operator()(int i, int j) { return a[i + static_cast<size_t>(j) * n]; }
  const C& operator()(int i, int j) const { return a[i + static_cast<size_t>(j) * n]; }
  static ZMat of(const double* p, int n) {
    ZMat m;
    m.n = n;
    m.a.assign(cptr(p), cptr(p) + static_cast<size_t>(n) * n);
    return m;
  }
  static ZMat identity(int n) {
    ZMat m;
    m.n = n;
    m.a.assign(static_cast<size_t>(n) * n, C(0));
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

ZMat mul(const ZMat& x, const ZMat& y) {
  const int n = x.n;
  ZMat r;
  r.n = n;
  r.a.assign(static_cast<size_t>(n) * n, C(0));
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const C b = y(k, j);
      if (b == C(0)) continue;
      for (int i = 0; i < n; ++i) r(i, j) += x(i, k) * b;
    }
  return r;
}
ZMat adjoint(const ZMat& x) {
  ZMat r = x;
  for (int j = 0; j < x.n; ++j)
    for (int i = 0; i < x.n; ++i) r(i, j) = std::conj(x(j, i));
  return r;
}
ZMat transpose(const ZMat& x) {
  ZMat r = x;
  for (int j = 0; j < x.n; ++j)
    for (int i = 0; i < x.n; ++i) r(i, j) = x(j, i);
  return r;
}
double fro(const ZMat& x) {
  double s = 0;
  for (const C& v : x.a) s += std::norm(v);
  return std::sqrt(s);
}
// exact structural test (matrix.hpp:152-172: LAPACK writes exact zeros)
bool upper(const ZMat& x) {
  for (int j = 0; j < x.n; ++j)
    for (int i = j + 1; i < x.n; ++i)
      if (x(i, j) != C(0)) return false;
  return true;
}

// Eigenbasis of an upper-triangular T: T P = P diag(T).  Column k solves
// (T_ii - T_kk) P_ik = -sum_{i<j<=k} T_ij P_jk upwards from P_kk = 1 and is
// scaled to unit 2-norm; P^{-1} by triangular back substitution.  A repeated
// eigenvalue with a non-zero coupling (defective T) gives kappa = inf.
struct Eig {
  ZMat P, Pinv;
  std::vector<C> lam;
  double kappa = std::numeric_limits<double>::infinity();
};
Eig eig_tri(const ZMat& T) {
  const int n = T.n;
  Eig e;
  e.P = ZMat::identity(n);
  e.lam.resize(n);
  for (int i = 0; i < n; ++i) e.lam[i] = T(i, i);
  for (int k = 0; k < n; ++k) {
    for (int i = k - 1; i >= 0; --i) {
      C num = 0;
      for (int j = i + 1; j <= k; ++j) num -= T(i, j) * e.P(j, k);
      const C den = T(i, i) - T(k, k);
      if (den == C(0)) {
        if (num != C(0)) return e;  // defective
        e.P(i, k) = 0;
      } else {
        e.P(i, k) = num / den;
      }
      if (!std::isfinite(std::abs(e.P(i, k)))) return e;
    }
    double s = 0;
    for (int i = 0; i <= k; ++i) s += std::norm(e.P(i, k));
    s = std::sqrt(s);
    for (int i = 0; i <= k; ++i) e.P(i, k) /= s;
  }
  // P^{-1}: upper triangular, column by column (P Y = I)
  e.Pinv = ZMat::identity(n);
  for (int k = 0; k < n; ++k)
    for (int i = k; i >= 0; --i) {
      C v = (i == k) ? C(1) : C(0);
      for (int j = i + 1; j <= k; ++j) v -= e.P(i, j) * e.Pinv(j, k);
      e.Pinv(i, k) = v / e.P(i, i);
    }
  e.kappa = fro(e.P) * fro(e.Pinv);
  if (!std::isfinite(e.kappa)) e.kappa = std::numeric_limits<double>::infinity();
  return e;
}

cudaError_t up(DevBuf& b, const C* h, size_t n) {
  if (cudaError_t e = b.ensure(2 * n); e != cudaSuccess) return e;
  return cudaMemcpy(b.p, h, n * sizeof(C), cudaMemcpyHostToDevice);
}

// One mode product on the device: the matrix (column-major) and its plain
// transpose (the NN operand of mode > 0).
struct DevOp {
  int mode = 0;
  DevBuf m, mt;
};
cudaError_t make_op(DevOp& op, int mode, const ZMat& M) {
  op.mode = mode;
  if (cudaError_t e = up(op.m, M.a.data(), M.a.size()); e != cudaSuccess) return e;
  const ZMat t = transpose(M);
  return up(op.mt, t.a.data(), t.a.size());
}

struct ZRun {
  tsg_ctx* ctx = nullptr;
  cudaStream_t st = nullptr;
  int d = 0;
  std::vector<int> dims;
  int64_t N = 0;
  double flops = 0;
  int launches = 0;
  DevBuf s1, s2;  // scratch of the operator chains

  // out = in x_{op_0} M_0 x_{op_1} M_1 ...  (out must differ from in unless
  // the chain is empty; in may be a scratch buffer only if it is s1 / s2)
  cudaError_t chain(const double* in, double* out, const std::vector<DevOp*>& ops) {
    if (ops.empty()) {
      if (in == out) return cudaSuccess;
      return cudaMemcpyAsync(out, in, N * sizeof(C), cudaMemcpyDeviceToDevice, st);
    }
    const double* cur = in;
    for (size_t k = 0; k < ops.size(); ++k) {
      double* dst = (k + 1 == ops.size()) ? out : (cur == s1.p ? s2.p : s1.p);
      if (cudaError_t e = tsg::zmode_product(cur, dst, d, dims.data(), ops[k]->mode, ops[k]->m.p,
                                             ops[k]->mt.p, dims[ops[k]->mode], 1.0, 0.0, st, &flops);
          e != cudaSuccess)
        return e;
      ++launches;
      cur = dst;
    }
    return cudaSuccess;
  }
};

// Test knob (read per call, like TSG_DECOUPLE at plan creation): force the
// reduced solve — 1 folded, 2 refined, 3 wavefront (Laplace); 0 = automatic.
int zpath_override() {
  const char* e = std::getenv("TSG_ZPATH");
  return e ? std::atoi(e) : 0;
}

// family 0 Laplace: T[0..d-1] triangular, U[m] unitary (NULL = reduced form).
// family 1 gsylv: T[0] = S, T[1..d-1] tails, Tc; U[0] = Q, Zb = Z (back of
// mode 0), U[1..] tail Schur vectors (all NULL = reduced form).
int zsolve(tsg_ctx* ctx, int family, int d, const int* dims, const double* const* T,
           const double* Tc, const double* const* U, const double* Zb, const double* B, double* X,
           const tsg_opts* opts, tsg_report* rep) {
  if (!ctx) return TSG_EINVAL;
  if (d < 2 || d > tsg::kZMaxOrder) return fail(ctx, TSG_EDIM, "order d must be in [2, 8]");
  if (!T || !B || !X) return fail(ctx, TSG_EDIM, "missing buffer");
  if (family == 1 && !Tc) return fail(ctx, TSG_EDIM, "gsylv needs the Tc factor");
  const bool reduced = (U == nullptr);
  int64_t N = 1;
  for (int m = 0; m < d; ++m) {
    if (dims[m] <= 0) return fail(ctx, TSG_EDIM, "dimensions must be positive");
    if (!T[m]) return fail(ctx, TSG_EDIM, "missing coefficient");
    if (!reduced && !U[m]) return fail(ctx, TSG_EDIM, "missing unitary factor");
    N *= dims[m];
  }
  if (family == 1 && !reduced && !Zb) return fail(ctx, TSG_EDIM, "missing Z factor");
  std::vector<ZMat> Tm(d);
  double scale = 0;
  for (int m = 0; m < d; ++m) {
    Tm[m] = ZMat::of(T[m], dims[m]);
    if (!upper(Tm[m]))
      return fail(ctx, TSG_EDIM, "coefficient " + std::to_string(m) + " must be upper triangular");
    scale += fro(Tm[m]);
  }
  ZMat Tcm;
  if (family == 1) {
    Tcm = ZMat::of(Tc, dims[0]);
    if (!upper(Tcm)) return fail(ctx, TSG_EDIM, "C must be upper triangular");
    scale += fro(Tcm);
  }
  const bool on_dev = opts && opts->inputs_on_device;

  // ---- choose the reduced solve
  std::vector<Eig> eg(d);
  int f = 0;
  if (family == 0) {
    for (int m = 0; m < d; ++m) eg[m] = eig_tri(Tm[m]);
    const int forced = opts ? opts->free_mode : -1;
    if (forced >= 0 && forced < d) {
      f = forced;
    } else {
      f = d - 1;
      for (int m = d - 1; m >= 0; --m)
        if (eg[m].kappa > eg[f].kappa) f = m;
    }
  } else {
    for (int m = 1; m < d; ++m) eg[m] = eig_tri(Tm[m]);
    f = 0;
  }
  double kprod = 1;
  for (int m = 0; m < d; ++m)
    if (m != f) kprod *= eg[m].kappa;
  enum Path { kFolded = 1, kRefined = 2, kWavefront = 3 };
  int path = kprod <= kFoldKappa ? kFolded : kprod <= kRefineKappa ? kRefined : kWavefront;
  if (family == 1 && path == kWavefront) path = kRefined;
  int refine_steps = kRefineSteps;
  if (family == 1 && !(kprod <= kRefineKappa)) refine_steps = 6;
  if (const int o = zpath_override(); o >= 1 && o <= 3 && !(o == kWavefront && family == 1) &&
                                      !(o != kWavefront && !std::isfinite(kprod)))
    path = o;

  TSG_CU(cudaSetDevice(ctx->device));
  ZRun run;
  run.ctx = ctx;
  run.st = ctx->stream;
  run.d = d;
  run.dims.assign(dims, dims + d);
  run.N = N;
  cudaStream_t st = run.st;

  // ---- device operators
  // Schur-basis transforms (absent for the reduced form)
  std::vector<DevOp> sfwd(reduced ? 0 : d), sback(reduced ? 0 : d);
  // eigenbasis changes (m != f), and folded transforms
  std::vector<DevOp> efwd(d), eback(d);
  std::vector<DevOp*> fwd_ops, back_ops, efwd_ops, eback_ops;
  for (int m = 0; m < d; ++m) {
    const bool dec = (path != kWavefront) && m != f;
    ZMat Sf, Sb;  // Schur transforms of this mode (identity when reduced)
    if (!reduced) {
      const ZMat Um = ZMat::of(U[m], dims[m]);
      Sf = adjoint(Um);  // gsylv mode 0: Q^H
      Sb = (family == 1 && m == 0) ? ZMat::of(Zb, dims[0]) : Um;
    }
    if (path == kFolded) {
      if (!dec && reduced) continue;
      const ZMat F = dec ? (reduced ? eg[m].Pinv : mul(eg[m].Pinv, Sf)) : Sf;
      const ZMat G = dec ? (reduced ? eg[m].P : mul(Sb, eg[m].P)) : Sb;
      TSG_CU(make_op(efwd[m], m, F));
      TSG_CU(make_op(eback[m], m, G));
      fwd_ops.push_back(&efwd[m]);
      back_ops.push_back(&eback[m]);
    } else {
      if (!reduced) {
        TSG_CU(make_op(sfwd[m], m, Sf));
        TSG_CU(make_op(sback[m], m, Sb));
        fwd_ops.push_back(&sfwd[m]);
        back_ops.push_back(&sback[m]);
      }
      if (dec) {
        TSG_CU(make_op(efwd[m], m, eg[m].Pinv));
        TSG_CU(make_op(eback[m], m, eg[m].P));
        efwd_ops.push_back(&efwd[m]);
        eback_ops.push_back(&eback[m]);
      }
    }
  }
  // fibre solve tables
  DevBuf dS, dTc, dScm, dTccm, dlam;
  tsg::ZFibreArgs fa{};
  tsg::ZLevelArgs la{};
  std::vector<DevBuf> dTt(d);
  const double tiny = std::numeric_limits<double>::epsilon() * 0.5 * scale;
  DevBuf dstatus;
  TSG_CU(dstatus.ensure(1));
  int* status = reinterpret_cast<int*>(dstatus.p);
  TSG_CU(cudaMemsetAsync(status, 0x7f, sizeof(int), st));
  if (path != kWavefront) {
    const ZMat St = transpose(family == 1 ? Tm[0] : Tm[f]);
    TSG_CU(up(dS, St.a.data(), St.a.size()));
    // column-major copies: operands of the blocked solve's GEMM updates
    const ZMat& Scm = family == 1 ? Tm[0] : Tm[f];
    TSG_CU(up(dScm, Scm.a.data(), Scm.a.size()));
    if (family == 1) {
      const ZMat Tct = transpose(Tcm);
      TSG_CU(up(dTc, Tct.a.data(), Tct.a.size()));
      TSG_CU(up(dTccm, Tcm.a.data(), Tcm.a.size()));
    }
    std::vector<C> lam;
    fa.x = nullptr;
    fa.d = d;
    fa.f = f;
    fa.nf = dims[f];
    int64_t sf = 1;
    for (int m = 0; m < d; ++m) {
      fa.dims[m] = dims[m];
      fa.lam_off[m] = static_cast<int>(lam.size());
      if (m != f) lam.insert(lam.end(), eg[m].lam.begin(), eg[m].lam.end());
      if (m < f) sf *= dims[m];
    }
    lam.push_back(0);
    TSG_CU(up(dlam, lam.data(), lam.size()));
    fa.sf = sf;
    fa.nfib = N / dims[f];
    fa.St = dS.p;
    fa.Tct = family == 1 ? dTc.p : nullptr;
    fa.S = dScm.p;
    fa.Tc = family == 1 ? dTccm.p : nullptr;
    fa.lam = dlam.p;
    fa.product = family;
    fa.tiny2 = tiny * tiny;
    fa.status = status;
  } else {
    la.d = d;
    int64_t s = 1;
    la.m0 = 0;
    for (int m = 0; m < d; ++m) {
      la.dims[m] = dims[m];
      la.stride[m] = s;
      s *= dims[m];
      if (dims[m] > dims[la.m0]) la.m0 = m;
      const ZMat t = transpose(Tm[m]);
      TSG_CU(up(dTt[m], t.a.data(), t.a.size()));
      la.Tt[m] = dTt[m].p;
    }
    la.nred = N / dims[la.m0];
    la.tiny2 = tiny * tiny;
    la.status = status;
  }
  // reduced-operator factors for the refinement residual (Schur basis)
  std::vector<DevOp> lop(d);
  DevOp lopc;
  if (path == kRefined) {
    for (int m = 0; m < d; ++m) TSG_CU(make_op(lop[m], m, Tm[m]));
    if (family == 1) TSG_CU(make_op(lopc, 0, Tcm));
  }

  // ---- buffers and timing
  DevBuf bt, xt, rr, dB, dX;
  DevBuf tmp, corr;  // refinement scratch: released with the others, after the last kernel
  TSG_CU(bt.ensure(2 * N));
  TSG_CU(xt.ensure(2 * N));
  TSG_CU(run.s1.ensure(2 * N));
  TSG_CU(run.s2.ensure(2 * N));
  if (path == kRefined) TSG_CU(rr.ensure(2 * N));
  const double* bin = B;
  double* xout = X;
  if (!on_dev) {
    TSG_CU(dB.ensure(2 * N));
    bin = dB.p;
    xout = bt.p;  // bt is free again once the back transforms start
  }
  cudaEvent_t* ev = ctx->ev;
  TSG_CU(cudaEventRecord(ev[0], st));
  if (!on_dev) TSG_CU(cudaMemcpyAsync(dB.p, B, N * sizeof(C), cudaMemcpyHostToDevice, st));
  TSG_CU(cudaEventRecord(ev[1], st));

  // dec(v -> out): eigenbasis changes, fibre solve, back (out != v)
  auto dec_solve = [&](const double* v, double* out) -> cudaError_t {
    if (cudaError_t e = run.chain(v, out, efwd_ops); e != cudaSuccess) return e;
    fa.x = out;
    fa.work = family == 1 ? run.s1.p : nullptr;  // the chains' scratch is idle during the solve
    if (cudaError_t e = tsg::zfibre_solve(fa, st, &run.launches, &run.flops); e != cudaSuccess) return e;
    if (eback_ops.empty()) return cudaSuccess;
    // back to the Schur basis through the scratch pair (out is neither)
    if (cudaError_t e = cudaMemcpyAsync(run.s2.p, out, N * sizeof(C), cudaMemcpyDeviceToDevice, st);
        e != cudaSuccess)
      return e;
    return run.chain(run.s2.p, out, eback_ops);
  };
  double* fwd_out = xt.p;
  if (path == kFolded) {
    TSG_CU(run.chain(bin, fwd_out, fwd_ops));
    TSG_CU(cudaEventRecord(ev[2], st));
    fa.x = fwd_out;
    fa.work = family == 1 ? run.s1.p : nullptr;  // the chains' scratch is idle during the solve
    TSG_CU(tsg::zfibre_solve(fa, st, &run.launches, &run.flops));
    TSG_CU(cudaEventRecord(ev[3], st));
    TSG_CU(run.chain(fwd_out, on_dev ? xout : bt.p, back_ops));
    xout = on_dev ? xout : bt.p;
  } else if (path == kWavefront) {
    TSG_CU(run.chain(bin, fwd_out, fwd_ops));
    TSG_CU(cudaEventRecord(ev[2], st));
    la.x = fwd_out;
    TSG_CU(tsg::zlevel_solve(la, st, &run.launches));
    TSG_CU(cudaEventRecord(ev[3], st));
    TSG_CU(run.chain(fwd_out, on_dev ? xout : bt.p, back_ops));
    xout = on_dev ? xout : bt.p;
  } else {
    // refined: b~ kept in bt (reduced: the input itself), x~ in xt
    const double* bref = bin;
    if (!fwd_ops.empty()) {
      TSG_CU(run.chain(bin, bt.p, fwd_ops));
      bref = bt.p;
    }
    TSG_CU(cudaEventRecord(ev[2], st));
    TSG_CU(tmp.ensure(2 * N));
    TSG_CU(corr.ensure(2 * N));
    TSG_CU(dec_solve(bref, xt.p));
    for (int k = 0; k < refine_steps; ++k) {
      // r = b~ - L(x~): copy b~, subtract the d (Laplace) or 2 (gsylv) terms
      TSG_CU(cudaMemcpyAsync(rr.p, bref, N * sizeof(C), cudaMemcpyDeviceToDevice, st));
      if (family == 0) {
        for (int m = 0; m < d; ++m) {
          TSG_CU(tsg::zmode_product(xt.p, rr.p, d, dims, m, lop[m].m.p, lop[m].mt.p, dims[m], -1.0,
                                    1.0, st, &run.flops));
          ++run.launches;
        }
      } else {
        TSG_CU(tsg::zmode_product(xt.p, rr.p, d, dims, 0, lop[0].m.p, lop[0].mt.p, dims[0], -1.0,
                                  1.0, st, &run.flops));
        std::vector<DevOp*> ch{&lopc};
        for (int m = 1; m < d; ++m) ch.push_back(&lop[m]);
        TSG_CU(run.chain(xt.p, tmp.p, ch));
        TSG_CU(tsg::axpy(rr.p, tmp.p, -1.0, 2 * N, st));
        run.launches += 2;
      }
      // x~ += dec(r)
      TSG_CU(dec_solve(rr.p, corr.p));
      TSG_CU(tsg::axpy(xt.p, corr.p, 1.0, 2 * N, st));
      ++run.launches;
    }
    TSG_CU(cudaEventRecord(ev[3], st));
    double* dst = on_dev ? xout : (bref == bt.p ? rr.p : bt.p);
    TSG_CU(run.chain(xt.p, dst, back_ops));
    xout = dst;
  }
  TSG_CU(cudaEventRecord(ev[4], st));
  if (!on_dev) TSG_CU(cudaMemcpyAsync(X, xout, N * sizeof(C), cudaMemcpyDeviceToHost, st));
  else if (xout != X) TSG_CU(cudaMemcpyAsync(X, xout, N * sizeof(C), cudaMemcpyDeviceToDevice, st));
  TSG_CU(cudaEventRecord(ev[5], st));
  int hstat = 0;
  TSG_CU(cudaMemcpyAsync(&hstat, status, sizeof(int), cudaMemcpyDeviceToHost, st));
  TSG_CU(cudaStreamSynchronize(st));
  if (rep) {
    float t = 0;
    *rep = tsg_report{};
    cudaEventElapsedTime(&t, ev[0], ev[1]);
    rep->t_h2d_ms = t;
    cudaEventElapsedTime(&t, ev[1], ev[2]);
    rep->t_fwd_ms = t;
    cudaEventElapsedTime(&t, ev[2], ev[3]);
    rep->t_solve_ms = t;
    cudaEventElapsedTime(&t, ev[3], ev[4]);
    rep->t_back_ms = t;
    cudaEventElapsedTime(&t, ev[4], ev[5]);
    rep->t_d2h_ms = t;
    cudaEventElapsedTime(&t, ev[0], ev[5]);
    rep->t_total_ms = t;
    // credited: complex transforms (8 N n per mode and direction) plus the
    // triangular applications (4 N (n_m - 1) real FLOP per mode)
    double sum_n = 0, sum_n1 = 0;
    for (int m = 0; m < d; ++m) {
      sum_n += dims[m];
      sum_n1 += dims[m] - 1;
    }
    rep->flops_alg = (reduced ? 0.0 : 16.0 * N * sum_n) + 4.0 * N * sum_n1;
    rep->flops_exec = run.flops;
    rep->zero_pivot_index = hstat == 0x7f7f7f7f ? -1 : hstat;
    rep->kernel_launches = run.launches;
  }
  if (hstat != 0x7f7f7f7f)
    return fail(ctx, TSG_ESINGULAR,
                "complex solve: numerically singular pivot (element/fibre " + std::to_string(hstat) +
                    ")");
  ctx->err = path == kFolded ? "zsolve: decoupled (folded)"
             : path == kRefined ? "zsolve: decoupled (refined)"
                                : "zsolve: wavefront";
  return TSG_OK;
}

}  // namespace

extern "C" {

int tsg_zlaplace_solve(tsg_ctx* ctx, int d, const int* dims, const double* const* T,
                       const double* const* U, const double* B, double* X, const tsg_opts* opts,
                       tsg_report* rep) {
  if (!U) return ctx ? fail(ctx, TSG_EDIM, "missing unitary factors") : TSG_EINVAL;
  return zsolve(ctx, 0, d, dims, T, nullptr, U, nullptr, B, X, opts, rep);
}

int tsg_zlaplace_reduced(tsg_ctx* ctx, int d, const int* dims, const double* const* T,
                         const double* Bt, double* Xt, const tsg_opts* opts, tsg_report* rep) {
  return zsolve(ctx, 0, d, dims, T, nullptr, nullptr, nullptr, Bt, Xt, opts, rep);
}

int tsg_zgsylv_solve(tsg_ctx* ctx, int d, const int* dims, const double* S, const double* Tc,
                     const double* Q, const double* Z, const double* const* Ttail,
                     const double* const* Utail, const double* B, double* X, const tsg_opts* opts,
                     tsg_report* rep) {
  if (!ctx) return TSG_EINVAL;
  if (d < 2 || d > tsg::kZMaxOrder) return fail(ctx, TSG_EDIM, "order d must be in [2, 8]");
  if (!Q || !Z || !Utail || !Ttail) return fail(ctx, TSG_EDIM, "missing factor");
  std::vector<const double*> t{S}, u{Q};
  for (int m = 1; m < d; ++m) {
    t.push_back(Ttail[m - 1]);
    u.push_back(Utail[m - 1]);
  }
  return zsolve(ctx, 1, d, dims, t.data(), Tc, u.data(), Z, B, X, opts, rep);
}

int tsg_zgsylv_reduced(tsg_ctx* ctx, int d, const int* dims, const double* S, const double* Tc,
                       const double* const* Ttail, const double* Bt, double* Xt,
                       const tsg_opts* opts, tsg_report* rep) {
  if (!ctx) return TSG_EINVAL;
  if (d < 2 || d > tsg::kZMaxOrder) return fail(ctx, TSG_EDIM, "order d must be in [2, 8]");
  if (!Ttail) return fail(ctx, TSG_EDIM, "missing factor");
  std::vector<const double*> t{S};
  for (int m = 1; m < d; ++m) t.push_back(Ttail[m - 1]);
  return zsolve(ctx, 1, d, dims, t.data(), Tc, nullptr, nullptr, Bt, Xt, opts, rep);
}

int tsg_zmode_multiply(tsg_ctx* ctx, int d, const int* dims, const double* X, int r,
                       const double* A, int mode, double* Y, const tsg_opts* opts) {
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
  std::vector<C> at(static_cast<size_t>(n) * r);
  const C* a = cptr(A);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < r; ++i) at[j + static_cast<size_t>(i) * n] = a[i + static_cast<size_t>(j) * r];
  DevBuf dx, dy, da, dat;
  TSG_CU(up(da, a, static_cast<size_t>(r) * n));
  TSG_CU(up(dat, at.data(), at.size()));
  const double* xin = X;
  double* yout = Y;
  if (!on_dev) {
    TSG_CU(up(dx, cptr(X), N));
    TSG_CU(dy.ensure(2 * NY));
    xin = dx.p;
    yout = dy.p;
  }
  TSG_CU(tsg::zmode_product(xin, yout, d, dims, mode, da.p, dat.p, r, 1.0, 0.0, st));
  if (!on_dev) TSG_CU(cudaMemcpyAsync(Y, dy.p, NY * sizeof(C), cudaMemcpyDeviceToHost, st));
  TSG_CU(cudaStreamSynchronize(st));
  return TSG_OK;
}

int tsg_zresidual(tsg_ctx* ctx, int family, int d, const int* dims, const double* const* A,
                  const double* Cm, const double* B, const double* X, int inputs_on_device,
                  double* out) {
  if (!ctx || !out) return TSG_EINVAL;
  if (d < 1 || d > TSG_MAX_ORDER) return fail(ctx, TSG_EDIM, "residual: order out of range");
  if (family == 1 && !Cm) return fail(ctx, TSG_EDIM, "residual: gsylv needs C");
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  int64_t N = 1;
  for (int m = 0; m < d; ++m) N *= dims[m];
  std::vector<DevOp> op(d);
  double scale = 0, prod = 1;
  for (int m = 0; m < d; ++m) {
    const ZMat a = ZMat::of(A[m], dims[m]);
    TSG_CU(make_op(op[m], m, a));
    const double f = fro(a);
    if (family == 0 || m == 0) scale += f;
    else prod *= f;
  }
  DevOp opc;
  if (family == 1) {
    const ZMat c = ZMat::of(Cm, dims[0]);
    TSG_CU(make_op(opc, 0, c));
    scale += fro(c) * prod;
  }
  DevBuf db, dx, r, acc;
  const double* b = B;
  const double* x = X;
  if (!inputs_on_device) {
    TSG_CU(up(db, cptr(B), N));
    TSG_CU(up(dx, cptr(X), N));
    b = db.p;
    x = dx.p;
  }
  TSG_CU(r.ensure(2 * N));
  TSG_CU(acc.ensure(3));
  TSG_CU(cudaMemcpyAsync(r.p, b, N * sizeof(C), cudaMemcpyDeviceToDevice, st));
  ZRun run;
  run.ctx = ctx;
  run.st = st;
  run.d = d;
  run.dims.assign(dims, dims + d);
  run.N = N;
  if (family == 0) {
    for (int m = 0; m < d; ++m)
      TSG_CU(tsg::zmode_product(x, r.p, d, dims, m, op[m].m.p, op[m].mt.p, dims[m], -1.0, 1.0, st));
  } else {
    TSG_CU(tsg::zmode_product(x, r.p, d, dims, 0, op[0].m.p, op[0].mt.p, dims[0], -1.0, 1.0, st));
    TSG_CU(run.s1.ensure(2 * N));
    TSG_CU(run.s2.ensure(2 * N));
    DevBuf t;
    TSG_CU(t.ensure(2 * N));
    std::vector<DevOp*> ch{&opc};
    for (int m = 1; m < d; ++m) ch.push_back(&op[m]);
    TSG_CU(run.chain(x, t.p, ch));
    TSG_CU(tsg::axpy(r.p, t.p, -1.0, 2 * N, st));
  }
  TSG_CU(cudaMemsetAsync(acc.p, 0, 3 * sizeof(double), st));
  TSG_CU(tsg::sumsq(r.p, 2 * N, acc.p, st));
  TSG_CU(tsg::sumsq(x, 2 * N, acc.p + 1, st));
  TSG_CU(tsg::sumsq(b, 2 * N, acc.p + 2, st));
  double h[3];
  TSG_CU(cudaMemcpyAsync(h, acc.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  TSG_CU(cudaStreamSynchronize(st));
  const double num = std::sqrt(h[0]), den = scale * std::sqrt(h[1]) + std::sqrt(h[2]);
  *out = den == 0 ? (num == 0 ? 0.0 : std::numeric_limits<double>::infinity()) : num / den;
  return TSG_OK;
}

}  // extern "C"
