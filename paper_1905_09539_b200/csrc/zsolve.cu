// Complex-scalar path: T = std::complex<double>
// problems and complex-triangular Schur arithmetic on sm_100a.
//
// Every buffer is interleaved (re, im) FP64 — the layout of the reference's
// std::vector<std::complex<double>> storage (tensor.hpp:19-27), so host
// tensors cross the C-ABI without a repacking pass.
//
//   zgemm_kernel        C[b] = alpha A[b] B[b] + beta C[b], complex, on FP64
//                       DMMA (four real m8n8k4 products per complex tile
//                       step: Cr += Ar Br - Ai Bi, Ci += Ar Bi + Ai Br).
//                       Replaces zgemm_ under mode_multiply<Complex>
//                       (tensor.hpp:187-231 -> blas.hpp:25-41).
//   zfibre_kernel       eigen-decoupled reduced solve: every mode but one
//                       (f) is in its eigenbasis, so each fibre along f is an
//                       independent triangular pencil system
//                       (S + z Tc) x = r with z = sum (Laplace) or product
//                       (gsylv) of the other modes' eigenvalues.
//   zlevel_kernel       robust fallback for Laplace operators whose
//                       eigenbases are too ill-conditioned to decouple: the
//                       reduced Kronecker sum of upper-triangular T_m is
//                       upper triangular, element i depends only on elements
//                       later in exactly one mode, so hyperplanes
//                       sum_m (n_m - 1 - i_m) = level are solved one launch
//                       each (the dependency DAG of lap_rec, laplace.hpp:
//                       134-153, flattened to its wavefronts).
#include <cstdint>

#include "common.cuh"
#include "util.h"
#include "zsolve.h"

namespace tsg {

namespace {

struct cplx {
  double r, i;
};
TSG_DEVINL cplx cmul(cplx a, cplx b) { return {a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
TSG_DEVINL cplx cadd(cplx a, cplx b) { return {a.r + b.r, a.i + b.i}; }
// a - b * c
TSG_DEVINL cplx cfms(cplx a, cplx b, cplx c) {
  return {fma(-b.i, -c.i, fma(-b.r, c.r, a.r)), fma(-b.r, c.i, fma(-b.i, c.r, a.i))};
}
TSG_DEVINL cplx ld2(const double* p) {
  const double2 v = *reinterpret_cast<const double2*>(p);
  return {v.x, v.y};
}
TSG_DEVINL void st2(double* p, cplx v) { *reinterpret_cast<double2*>(p) = make_double2(v.r, v.i); }
TSG_DEVINL double neg(double x) {
  return __longlong_as_double(__double_as_longlong(x) ^ static_cast<long long>(0x8000000000000000ULL));
}

// ---------------------------------------------------------------------------
// zgemm: CTA tile 64 x 64 complex, k-step 8 complex, four warps of 32 x 32
// complex (4 x 4 fragments of 8 x 8, two accumulators each), 3-stage
// cp.async ring.  Shared tiles keep the interleaved layout; fragments are
// read as double2 (LDS.128): A stage [BK][LDA] with LDA = 2 BM + 4 doubles
// and B stage [BN][LDB] with LDB = 2 BK + 8 doubles make every quarter-warp
// (2 x 4 lanes) hit eight distinct 16-byte bank groups.
constexpr int ZBM = 64, ZBN = 64, ZBK = 8, ZST = 3, ZNT = 128;
constexpr int ZLDA = 2 * ZBM + 4, ZLDB = 2 * ZBK + 8;
constexpr int ZA_ELEMS = ZBK * ZLDA, ZB_ELEMS = ZBN * ZLDB, ZSTAGE = ZA_ELEMS + ZB_ELEMS;
constexpr int ZSMEM = ZST * ZSTAGE * 8;

__global__ void __launch_bounds__(ZNT, 2) zgemm_kernel(ZGemmArgs g) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int gq = lane >> 2, tq = lane & 3;
  const int64_t tiles_m = (g.M + ZBM - 1) / ZBM, tiles_n = (g.N + ZBN - 1) / ZBN;
  const int64_t bid = blockIdx.x;
  const int m0 = static_cast<int>((bid % tiles_m) * ZBM);
  const int n0 = static_cast<int>(((bid / tiles_m) % tiles_n) * ZBN);
  const int64_t bt = bid / (tiles_m * tiles_n);
  const double* __restrict__ A = g.A + 2 * bt * g.sA;
  const double* __restrict__ B = g.B + 2 * bt * g.sB;
  double* __restrict__ C = g.C + 2 * bt * g.sC;

  auto load_stage = [&](int stage, int k0) {
    double* sa = smem + stage * ZSTAGE;
    double* sb = sa + ZA_ELEMS;
#pragma unroll
    for (int c = tid; c < ZBK * ZBM; c += ZNT) {
      const int kk = c / ZBM, mm = c % ZBM;
      const int gm = m0 + mm, gk = k0 + kk;
      const bool ok = gm < g.M && gk < g.K;
      cp_async16(sa + kk * ZLDA + 2 * mm, ok ? A + 2 * (static_cast<int64_t>(gk) * g.lda + gm) : A,
                 ok ? 16 : 0);
    }
#pragma unroll
    for (int c = tid; c < ZBN * ZBK; c += ZNT) {
      const int nn = c / ZBK, kk = c % ZBK;
      const int gn = n0 + nn, gk = k0 + kk;
      const bool ok = gn < g.N && gk < g.K;
      cp_async16(sb + nn * ZLDB + 2 * kk, ok ? B + 2 * (static_cast<int64_t>(gn) * g.ldb + gk) : B,
                 ok ? 16 : 0);
    }
  };

  double accr[4][4][2], acci[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) accr[i][j][0] = accr[i][j][1] = acci[i][j][0] = acci[i][j][1] = 0.0;

  const int nk = (g.K + ZBK - 1) / ZBK;
#pragma unroll
  for (int s = 0; s < ZST - 1; ++s) {
    if (s < nk) load_stage(s, s * ZBK);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<ZST - 2>();
    __syncthreads();
    {
      const int nxt = kt + ZST - 1;
      if (nxt < nk) load_stage(nxt % ZST, nxt * ZBK);
      cp_async_commit();
    }
    const double* sa = smem + (kt % ZST) * ZSTAGE;
    const double* sb = sa + ZA_ELEMS;
#pragma unroll
    for (int k4 = 0; k4 < ZBK; k4 += 4) {
      double ar[4], ai[4], an[4], br[4], bi[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double2 v =
            *reinterpret_cast<const double2*>(sa + (k4 + tq) * ZLDA + 2 * (wm * 32 + i * 8 + gq));
        ar[i] = v.x;
        ai[i] = v.y;
        an[i] = neg(v.y);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 v =
            *reinterpret_cast<const double2*>(sb + (wn * 32 + j * 8 + gq) * ZLDB + 2 * (k4 + tq));
        br[j] = v.x;
        bi[j] = v.y;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma(accr[i][j][0], accr[i][j][1], ar[i], br[j]);
          dmma(acci[i][j][0], acci[i][j][1], ar[i], bi[j]);
          dmma(accr[i][j][0], accr[i][j][1], an[i], bi[j]);
          dmma(acci[i][j][0], acci[i][j][1], ai[i], br[j]);
        }
    }
  }
  cp_async_wait_all();

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + gq;
    if (row >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * 32 + j * 8 + 2 * tq + h;
        if (col >= g.N) continue;
        double* p = C + 2 * (static_cast<int64_t>(col) * g.ldc + row);
        cplx v{g.alpha * accr[i][j][h], g.alpha * acci[i][j][h]};
        if (g.beta != 0.0) {
          const cplx o = ld2(p);
          v.r = fma(g.beta, o.r, v.r);
          v.i = fma(g.beta, o.i, v.i);
        }
        st2(p, v);
      }
  }
}

// ---------------------------------------------------------------------------
// Decoupled fibre solve, diagonal block rows [i_lo, i_hi) (<= ZFB rows) of
// every fibre along mode f: thread = one fibre, a CTA stages the block rows of
// its ZFT fibres in shared memory (coalesced: rows of f > 0 are contiguous
// across fibres, fibres of f = 0 are contiguous along the rows), substitutes
// them bottom-up (the rows below the block were applied by the GEMM updates
// of zfibre_solve; the row-major S / Tc rows are read by every lane at the
// same address) and writes x back — for gsylv also z x into `work`, the
// operand of the Tc updates of the blocks above.
constexpr int ZFB = 32;         // rows per diagonal block
constexpr int ZFT = 128;        // fibres per CTA
constexpr int ZFP = ZFB + 1;    // shared pitch (complex elements) per fibre
constexpr int ZFSMEM = ZFT * ZFP * 2 * static_cast<int>(sizeof(double));

__global__ void __launch_bounds__(ZFT) zfibre_kernel(const ZFibreArgs a) {
  extern __shared__ __align__(16) double zsm[];
  const int64_t q0 = blockIdx.x * static_cast<int64_t>(ZFT);
  const int nfib = static_cast<int>(a.nfib - q0 < ZFT ? a.nfib - q0 : ZFT);
  const int n = a.nf, lo_r = a.i_lo, nr = a.i_hi - a.i_lo;
  const int64_t sf = a.sf;
  // element (fibre q, row i): x + 2 * ((q % sf) + i * sf + (q / sf) * sf * n)
  auto fibre_base = [&](int64_t q) { return (q % sf) + (q / sf) * sf * n; };
  if (a.f == 0) {  // sf == 1: a fibre's rows are contiguous
    for (int e = threadIdx.x; e < nfib * nr; e += ZFT) {
      const int t = e / nr, i = e - t * nr;
      st2(zsm + 2 * (t * ZFP + i), ld2(a.x + 2 * ((q0 + t) * n + lo_r + i)));
    }
  } else if (threadIdx.x < nfib) {
    const double* xp = a.x + 2 * (fibre_base(q0 + threadIdx.x) + lo_r * sf);
    for (int i = 0; i < nr; ++i) st2(zsm + 2 * (threadIdx.x * ZFP + i), ld2(xp + 2 * i * sf));
  }
  __syncthreads();
  if (threadIdx.x < nfib) {
    const int64_t q = q0 + threadIdx.x;
    const int64_t lo = q % sf, hi = q / sf;
    // the other modes' eigenvalues combine into z
    cplx z = a.product ? cplx{1.0, 0.0} : cplx{0.0, 0.0};
    int64_t r = lo;
    for (int m = 0; m < a.f; ++m) {
      const int i = static_cast<int>(r % a.dims[m]);
      r /= a.dims[m];
      const cplx l = ld2(a.lam + 2 * (a.lam_off[m] + i));
      z = a.product ? cmul(z, l) : cadd(z, l);
    }
    r = hi;
    for (int m = a.f + 1; m < a.d; ++m) {
      const int i = static_cast<int>(r % a.dims[m]);
      r /= a.dims[m];
      const cplx l = ld2(a.lam + 2 * (a.lam_off[m] + i));
      z = a.product ? cmul(z, l) : cadd(z, l);
    }
    double* xs = zsm + 2 * (threadIdx.x * ZFP);
    for (int i = nr - 1; i >= 0; --i) {
      cplx acc = ld2(xs + 2 * i);
      const double* srow = a.St + 2 * (static_cast<int64_t>(lo_r + i) * n + lo_r);
      const double* trow = a.Tct ? a.Tct + 2 * (static_cast<int64_t>(lo_r + i) * n + lo_r) : nullptr;
      for (int j = i + 1; j < nr; ++j) {
        cplx c = ld2(srow + 2 * j);
        if (trow) c = cadd(c, cmul(z, ld2(trow + 2 * j)));
        acc = cfms(acc, c, ld2(xs + 2 * j));
      }
      cplx dg = ld2(srow + 2 * i);
      dg = trow ? cadd(dg, cmul(z, ld2(trow + 2 * i))) : cadd(dg, z);
      const double m2 = dg.r * dg.r + dg.i * dg.i;
      if (!(m2 > a.tiny2)) {
        atomicMin(a.status, static_cast<int>(q < 0x7fffffff ? q : 0x7ffffffe));
        st2(xs + 2 * i, {0.0, 0.0});
        continue;
      }
      const double inv = 1.0 / m2;
      st2(xs + 2 * i, {(acc.r * dg.r + acc.i * dg.i) * inv, (acc.i * dg.r - acc.r * dg.i) * inv});
    }
    if (a.work && a.i_lo > 0) {  // z x for the Tc updates of the blocks above (f = 0)
      double* wp = a.work + 2 * (q * n + lo_r);
      for (int i = 0; i < nr; ++i) st2(wp + 2 * i, cmul(z, ld2(xs + 2 * i)));
    }
  }
  __syncthreads();
  if (a.f == 0) {
    for (int e = threadIdx.x; e < nfib * nr; e += ZFT) {
      const int t = e / nr, i = e - t * nr;
      st2(a.x + 2 * ((q0 + t) * n + lo_r + i), ld2(zsm + 2 * (t * ZFP + i)));
    }
  } else if (threadIdx.x < nfib) {
    double* xp = a.x + 2 * (fibre_base(q0 + threadIdx.x) + lo_r * sf);
    for (int i = 0; i < nr; ++i) st2(xp + 2 * i * sf, ld2(zsm + 2 * (threadIdx.x * ZFP + i)));
  }
}

// ---------------------------------------------------------------------------
// Wavefront level of the fully triangular reduced Laplace solve: the threads
// enumerate every mode but m0 (m0 fastest-varying excluded), i_m0 follows
// from the level.  x holds B~ on entry and is overwritten in place; every
// element read besides the own one lies on an earlier level.
__global__ void __launch_bounds__(128) zlevel_kernel(const ZLevelArgs a) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= a.nred) return;
  int idx[kZMaxOrder];
  int64_t r = q;
  int s = 0;
  for (int m = 0; m < a.d; ++m) {
    if (m == a.m0) continue;
    idx[m] = static_cast<int>(r % a.dims[m]);
    r /= a.dims[m];
    s += a.dims[m] - 1 - idx[m];
  }
  const int l0 = a.level - s;
  if (l0 < 0 || l0 >= a.dims[a.m0]) return;
  idx[a.m0] = a.dims[a.m0] - 1 - l0;
  int64_t e = 0;
  for (int m = 0; m < a.d; ++m) e += idx[m] * a.stride[m];
  cplx acc = ld2(a.x + 2 * e);
  cplx dg{0.0, 0.0};
  for (int m = 0; m < a.d; ++m) {
    const int n = a.dims[m], i = idx[m];
    const double* row = a.Tt[m] + 2 * static_cast<int64_t>(i) * n;
    dg = cadd(dg, ld2(row + 2 * i));
    const double* xm = a.x + 2 * (e - i * a.stride[m]);
    const int64_t s2 = 2 * a.stride[m];
    for (int j = i + 1; j < n; ++j) acc = cfms(acc, ld2(row + 2 * j), ld2(xm + j * s2));
  }
  const double m2 = dg.r * dg.r + dg.i * dg.i;
  if (!(m2 > a.tiny2)) {
    atomicMin(a.status, static_cast<int>(e < 0x7fffffff ? e : 0x7ffffffe));
    st2(a.x + 2 * e, {0.0, 0.0});
    return;
  }
  const double inv = 1.0 / m2;
  st2(a.x + 2 * e, {(acc.r * dg.r + acc.i * dg.i) * inv, (acc.i * dg.r - acc.r * dg.i) * inv});
}

}  // namespace

cudaError_t zgemm(const ZGemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return cudaSuccess;
  const int64_t tiles = ((g.M + ZBM - 1) / ZBM) * ((g.N + ZBN - 1) / ZBN) * g.batch;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidValue;
  int nsm = 0, occ = 0;
  if (cudaError_t e = kernel_setup(zgemm_kernel, ZSMEM, ZNT, &nsm, &occ); e != cudaSuccess) return e;
  zgemm_kernel<<<static_cast<unsigned>(tiles), ZNT, ZSMEM, st>>>(g);
  return cudaGetLastError();
}

cudaError_t zmode_product(const double* X, double* Y, int d, const int* dims, int mode,
                          const double* A, const double* At, int r, double alpha, double beta,
                          cudaStream_t st, double* flops) {
  int64_t P = 1, Q = 1;
  for (int v = 0; v < mode; ++v) P *= dims[v];
  for (int v = mode + 1; v < d; ++v) Q *= dims[v];
  const int n = dims[mode];
  ZGemmArgs g{};
  g.alpha = alpha;
  g.beta = beta;
  if (mode == 0) {
    // Y_(0) (r x Q) = A (r x n) X_(0) (n x Q)           (tensor.hpp:203-210)
    if (Q > 0x7fffffffLL) return cudaErrorInvalidValue;
    g.A = A;
    g.B = X;
    g.C = Y;
    g.M = r;
    g.N = static_cast<int>(Q);
    g.K = n;
    g.lda = r;
    g.ldb = n;
    g.ldc = r;
    g.batch = 1;
  } else {
    // per slab q: Y_q (P x r) = X_q (P x n) A^T (n x r)  (tensor.hpp:211-229)
    if (P > 0x7fffffffLL) return cudaErrorInvalidValue;
    g.A = X;
    g.B = At;
    g.C = Y;
    g.M = static_cast<int>(P);
    g.N = r;
    g.K = n;
    g.lda = P;
    g.ldb = n;
    g.ldc = P;
    g.sA = P * n;
    g.sC = P * r;
    g.batch = Q;
  }
  if (flops) *flops += 8.0 * static_cast<double>(P) * Q * n * r;
  return zgemm(g, st);
}

cudaError_t zfibre_solve(const ZFibreArgs& a0, cudaStream_t st, int* launches, double* flops) {
  if (a0.nfib <= 0 || a0.nf <= 0) return cudaSuccess;
  ZFibreArgs a = a0;
  const int n = a.nf;
  const bool gs = a.Tct != nullptr;
  // blocked only with the operands of the GEMM updates at hand
  const bool blocked = n > ZFB && (a.f > 0 || a.S) && (!gs || (a.f == 0 && a.Tc && a.work));
  if (!blocked && n > ZFB) return cudaErrorInvalidValue;
  if (gs && a.f != 0) return cudaErrorInvalidValue;
  int nsm = 0, occ = 0;
  if (cudaError_t e = kernel_setup(zfibre_kernel, ZFSMEM, ZFT, &nsm, &occ); e != cudaSuccess) return e;
  const int64_t blocks = (a.nfib + ZFT - 1) / ZFT;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int64_t P = a.sf, Q = a.nfib / a.sf;
  for (int hi = n; hi > 0;) {
    const int lo = hi > ZFB ? hi - ZFB : 0;
    if (hi < n) {
      // x[lo:hi] -= S[lo:hi, hi:n] x[hi:n]  (+ Tc[lo:hi, hi:n] (z x)[hi:n])
      ZGemmArgs g{};
      g.alpha = -1.0;
      g.beta = 1.0;
      g.K = n - hi;
      if (a.f == 0) {
        if (Q > 0x7fffffffLL) return cudaErrorInvalidValue;
        g.M = hi - lo;
        g.N = static_cast<int>(Q);
        g.lda = g.ldb = g.ldc = n;
        g.batch = 1;
        g.A = a.S + 2 * (lo + static_cast<int64_t>(hi) * n);
        g.B = a.x + 2 * static_cast<int64_t>(hi);
        g.C = a.x + 2 * static_cast<int64_t>(lo);
        if (cudaError_t e = zgemm(g, st); e != cudaSuccess) return e;
        if (gs) {
          g.A = a.Tc + 2 * (lo + static_cast<int64_t>(hi) * n);
          g.B = a.work + 2 * static_cast<int64_t>(hi);
          if (cudaError_t e = zgemm(g, st); e != cudaSuccess) return e;
        }
      } else {
        // per slab: X_q[:, lo:hi] -= X_q[:, hi:n] (S[lo:hi, hi:n])^T; St is S^T column-major
        if (P > 0x7fffffffLL) return cudaErrorInvalidValue;
        g.M = static_cast<int>(P);
        g.N = hi - lo;
        g.lda = g.ldc = P;
        g.ldb = n;
        g.sA = g.sC = P * n;
        g.sB = 0;
        g.batch = Q;
        g.A = a.x + 2 * (static_cast<int64_t>(hi) * P);
        g.B = a.St + 2 * (hi + static_cast<int64_t>(lo) * n);
        g.C = a.x + 2 * (static_cast<int64_t>(lo) * P);
        if (cudaError_t e = zgemm(g, st); e != cudaSuccess) return e;
      }
      if (launches) *launches += gs ? 2 : 1;
      if (flops) *flops += (gs ? 16.0 : 8.0) * static_cast<double>(a.nfib) * (hi - lo) * (n - hi);
    }
    a.i_lo = lo;
    a.i_hi = hi;
    zfibre_kernel<<<static_cast<unsigned>(blocks), ZFT, ZFSMEM, st>>>(a);
    if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
    if (launches) *launches += 1;
    hi = lo;
  }
  return cudaSuccess;
}

cudaError_t zlevel_solve(ZLevelArgs a, cudaStream_t st, int* launches) {
  int levels = 1;
  for (int m = 0; m < a.d; ++m) levels += a.dims[m] - 1;
  const int64_t blocks = (a.nred + 127) / 128;
  for (int l = 0; l < levels; ++l) {
    a.level = l;
    zlevel_kernel<<<static_cast<unsigned>(blocks), 128, 0, st>>>(a);
    if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
  }
  if (launches) *launches += levels;
  return cudaSuccess;
}

}  // namespace tsg
