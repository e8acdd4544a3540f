// Generalised Sylvester (gsylv, family 1) reduced solve for d = 3..5 (C5:
// 200 x 40^3): the small-tile dataflow of solve_lapd.cu with the chain
// factorisation of the Kronecker product term.
//
// Reduced equation (gsylv.hpp:62-159):
//   X x_0 S + (X x_1 A_1 ... x_{d-1} A_{d-1}) x_0 Tc = B~
// with S quasi-upper (QZ), Tc upper triangular, A_m quasi-upper (Schur).
// The product term is the chain W_{d-1} = X x_{d-1} A_{d-1},
// W_m = W_{m+1} x_m A_m, V = W_1 (gsylv.hpp:111-123), so every tile of W_m
// depends on W_{m+1} tiles later along mode m only.  Per tile t:
//   1. gather B~_t; L_m = sum_{s > t_m} A_m[t_m, s] x_m W_{m+1}(t|m->s)
//      (W_d = X) and the mode-0 terms B~_t -= sum_{s > t_0} S[t_0, s] X_s +
//      Tc[t_0, s] V_s, on DMMA with the source tensor as the A operand
//      (solve_lapd.cu), far tiles (>= t+2) first, then t+1;
//   2. V_t = K_tt X_t + R_t with K_tt = (x)_m A_m,tt and
//      R = A_1 (A_2 (... L_{d-1}) + L_2) + L_1, so the tile equation is
//      S_tt X + Tc_tt (K_tt X) = B~_t - Tc_tt R;
//   3. base case: diagonalise the tail blocks (complex bases V_m of the
//      tile's Schur blocks, host tables), then for every tail eigen-index j
//      solve the e_0 x e_0 quasi-triangular pencil (S_tt + z_j Tc_tt) x = r,
//      z_j = prod_m lambda_m(j_m), by back substitution over the Schur cells
//      of S (one thread per mode-0 fibre); back to the Schur basis;
//   4. W_{d-1} = A_{d-1,tt} X_t + L_{d-1}, W_m = A_m,tt W_{m+1} + L_m;
//      store X_t and W_m(t), release.
// Reference: gs_rec / gsylv_base (gsylv.hpp:70-128), gsylv_merged base
// (gsylv.hpp:167-232), block_back_substitution (kernels.hpp:179-261).
#include <cstdint>

#include "common.cuh"
#include "solve.h"
#include "util.h"

namespace tsg {
namespace {

constexpr int THREADS = 128, WARPS = 4, EP = 512;
constexpr int VHS = kVhStride;
constexpr int NBMAX = EP / 2 / 8 / WARPS;

template <int D>
struct GG {
  int64_t lt, gbase;
  int start[D], ext[D], tco[D];
  unsigned char rk[8];  // mode-0 rows: 0 1x1 cell, 1/2 first/second row of a 2x2 cell
};

TSG_DEVINL void waitg(const SolveArgs& a, int64_t tile) {
  const int* f = a.flags + tile;
  unsigned ns = 32;
  while (ld_acquire(f) < a.epoch) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
}

// dst += sign * sum_k src(cross, k) Tm(rows, k) over rows k in [klo, khi).
// NB 8-column blocks per warp and round, UB k4-steps of loads in flight
// (NB * UB <= 16 fragment loads per batch).
template <int D, int NB, int UB>
TSG_DEVINL void update_nb(const SolveArgs& a, const GG<D>& g, double* dst, const int64_t* goff, double sign, int ep,
                          int m, int klo, int khi, const double* Tm, const double* src) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int lpm = a.tlog[m], shm = a.tsh[m];
  const int cross = ep >> lpm;
  const int nblk = (cross + 7) >> 3;
  const int nm = a.dims[m];
  const int64_t sm = a.stride[m];
  const int row = g.start[m] + gq;
  const bool rok = gq < g.ext[m];
  // src(cross n, k) = src[goff[lt(n)] + (k - start_m) * stride_m] (goff < 0:
  // padded cross column, skipped); lt(n) inserts mode m's zero bit field
  const int64_t kofs = static_cast<int64_t>(klo + tq - g.start[m]) * sm;
  const int64_t s4 = 4 * sm;
  const double* pt0 = Tm + row + static_cast<int64_t>(klo + tq) * nm;
  const int64_t t4 = 4 * static_cast<int64_t>(nm);
  for (int base = warp; base < nblk; base += WARPS * NB) {
    int ltc[NB];
    const double* px[NB];
    bool cok[NB];
    double acc[NB][2];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int b = base + WARPS * j;
      const int n = 8 * b + gq;
      acc[j][0] = acc[j][1] = 0.0;
      ltc[j] = (n & ((1 << shm) - 1)) | ((n >> shm) << (shm + lpm));
      const int64_t go = (b < nblk && n < cross) ? goff[ltc[j]] : -1;
      cok[j] = go >= 0;
      px[j] = src + (cok[j] ? go + kofs : 0);
    }
    const double* pt = pt0;
    for (int k0 = klo; k0 < khi; k0 += 4 * UB) {
      double bt[UB], av[UB][NB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const bool kok = k0 + 4 * u + tq < khi;
        bt[u] = (kok && rok) ? __ldg(pt + u * t4) : 0.0;
#pragma unroll
        for (int j = 0; j < NB; ++j) av[u][j] = (cok[j] && kok) ? ld_cg(px[j] + u * s4) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UB; ++u)
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (base + WARPS * j < nblk) dmma(acc[j][0], acc[j][1], av[u][j], bt[u]);
      pt += UB * t4;
#pragma unroll
      for (int j = 0; j < NB; ++j) px[j] += UB * s4;
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      if (!cok[j]) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 2 * tq + h;
        if (r < (1 << lpm)) dst[ltc[j] + (r << shm)] += sign * acc[j][h];
      }
    }
  }
}

template <int D>
TSG_DEVINL void update_src(const SolveArgs& a, const GG<D>& g, double* dst, const int64_t* goff, double sign,
                           int ep, int m, int klo, int khi, const double* Tm, const double* src) {
  const int nblk = ((ep >> a.tlog[m]) + 7) >> 3;
  if (nblk <= 2 * WARPS) update_nb<D, 2, 8>(a, g, dst, goff, sign, ep, m, klo, khi, Tm, src);
  else if (nblk <= 4 * WARPS) update_nb<D, 4, 4>(a, g, dst, goff, sign, ep, m, klo, khi, Tm, src);
  else update_nb<D, 8, 2>(a, g, dst, goff, sign, ep, m, klo, khi, Tm, src);
}

// tile-local offset of the first element of fibre f along mode m (the
// tile index concatenates the modes' bit fields: insert mode m's zero field)
template <int D>
TSG_DEVINL int fibre_lt(const SolveArgs& a, int m, int f) {
  const int sh = a.tsh[m];
  return (f & ((1 << sh) - 1)) | ((f >> sh) << (sh + a.tlog[m]));
}

// buf(fibre along m) = add(fibre) + sign * M (P x P of a row-major stride-8
// block) buf(fibre), P the padded extent of mode m (compile time)
template <int D, int P>
TSG_DEVINL void rmode_p(const SolveArgs& a, double* buf, const double* add, const double* M, int ep, int m,
                        double sign, const double* src = nullptr) {
  // buf(fibre) = add(fibre) + sign M src(fibre), src = buf when null
  const int shm = a.tsh[m];
  const double* in = src ? src : buf;
  for (int f = threadIdx.x; f < ep / P; f += THREADS) {
    const int lt0 = fibre_lt<D>(a, m, f);
    double x[P];
#pragma unroll
    for (int r = 0; r < P; ++r) x[r] = in[lt0 + (r << shm)];
#pragma unroll
    for (int r = 0; r < P; ++r) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < P; ++c) s = fma(M[8 * r + c], x[c], s);
      const int l = lt0 + (r << shm);
      buf[l] = (add ? add[l] : 0.0) + sign * s;
    }
  }
}

template <int D>
TSG_DEVINL void rmode(const SolveArgs& a, const GG<D>& g, double* buf, const double* add, const double* M,
                      int ep, int m, double sign = 1.0, const double* src = nullptr) {
  switch (a.tlog[m]) {
    case 0: rmode_p<D, 1>(a, buf, add, M, ep, m, sign, src); break;
    case 1: rmode_p<D, 2>(a, buf, add, M, ep, m, sign, src); break;
    case 2: rmode_p<D, 4>(a, buf, add, M, ep, m, sign, src); break;
    default: rmode_p<D, 8>(a, buf, add, M, ep, m, sign, src); break;
  }
}

// complex mode product with an 8x8 table (re at Vr, im at Vr + 64)
template <int D, int P>
TSG_DEVINL void cmode_p(const SolveArgs& a, double* xr, double* xi, const double* Vr, int ep, int m) {
  const int shm = a.tsh[m];
  const double* Vi = Vr + 64;
  for (int f = threadIdx.x; f < ep / P; f += THREADS) {
    const int lt0 = fibre_lt<D>(a, m, f);
    double zr[P], zi[P];
#pragma unroll
    for (int r = 0; r < P; ++r) {
      zr[r] = xr[lt0 + (r << shm)];
      zi[r] = xi[lt0 + (r << shm)];
    }
#pragma unroll
    for (int r = 0; r < P; ++r) {
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int c = 0; c < P; ++c) {
        const double ar = Vr[8 * r + c], ai = Vi[8 * r + c];
        sr = fma(ar, zr[c], fma(-ai, zi[c], sr));
        si = fma(ar, zi[c], fma(ai, zr[c], si));
      }
      xr[lt0 + (r << shm)] = sr;
      xi[lt0 + (r << shm)] = si;
    }
  }
}

template <int D>
TSG_DEVINL void cmode(const SolveArgs& a, const GG<D>& g, double* xr, double* xi, const double* Vr, int ep,
                      int m) {
  switch (a.tlog[m]) {
    case 0: cmode_p<D, 1>(a, xr, xi, Vr, ep, m); break;
    case 1: cmode_p<D, 2>(a, xr, xi, Vr, ep, m); break;
    case 2: cmode_p<D, 4>(a, xr, xi, Vr, ep, m); break;
    default: cmode_p<D, 8>(a, xr, xi, Vr, ep, m); break;
  }
}

template <int D>
#ifndef GSYD_MINB
#define GSYD_MINB 3
#endif
__global__ void __launch_bounds__(THREADS, GSYD_MINB) solve_gsyd_kernel(SolveArgs a) {
  __shared__ __align__(16) double xr[EP];
  __shared__ __align__(16) double xi[EP];
  __shared__ __align__(16) double lb[D - 1][EP];  // L_m -> W_m (m = 1..D-1)
  __shared__ __align__(16) double rb[EP];         // R chain
  __shared__ __align__(16) double vh[(D - 1) * VHS];
  __shared__ double blk[D + 1][64];                // S_tt, A_m,tt (m >= 1), Tc_tt: 8x8 row-major
  __shared__ int64_t goff[EP];                     // global offset per tile element (-1: padding)
  __shared__ GG<D> g;
  __shared__ int s_tile;
  const int tid = threadIdx.x;
  int ep = 1;
#pragma unroll
  for (int m = 0; m < D; ++m) ep <<= a.tlog[m];

  for (;;) {
    if (tid == 0) s_tile = atomicAdd(a.counter, 1);
    __syncthreads();
    const int qi = s_tile;
    if (qi >= a.ntiles) break;
    if (tid < D) {
      const unsigned long long pk = a.ocoord[qi];
      const int tm = static_cast<int>((pk >> (10 * tid)) & 1023);
      const TileMode& src = a.tmode[tid][tm];
      g.tco[tid] = tm;
      g.start[tid] = src.start;
      g.ext[tid] = src.ext;
      if (tid == 0) {
        g.lt = a.order[qi];
        for (int k = 0; k < 8; ++k) g.rk[k] = 0;
        for (int c = 0; c < src.nc; ++c)
          if (src.cz[c] == 2 && src.cs[c] + 1 < 8) {
            g.rk[src.cs[c]] = 1;
            g.rk[src.cs[c] + 1] = 2;
          }
      }
    }
    __syncthreads();
    if (tid == 0) {
      int64_t gb = 0;
      for (int m = 0; m < D; ++m) gb += static_cast<int64_t>(g.start[m]) * a.stride[m];
      g.gbase = gb;
    }
    __syncthreads();

    // ---- gather B~_t, tables, diagonal blocks; zero the chain buffers ----
    for (int l = tid; l < ep; l += THREADS) {
      int64_t off = g.gbase;
      bool ok = true;
#pragma unroll
      for (int v = 0; v < D; ++v) {
        const int iv = (l >> a.tsh[v]) & ((1 << a.tlog[v]) - 1);
        ok &= iv < g.ext[v];
        off += static_cast<int64_t>(iv) * a.stride[v];
      }
      cp_async8(xr + l, ok ? a.X + off : a.X, ok ? 8 : 0);
      xi[l] = 0.0;
      goff[l] = ok ? off : -1;
#pragma unroll
      for (int m = 0; m < D - 1; ++m) lb[m][l] = 0.0;
    }
#pragma unroll
    for (int m = 1; m < D; ++m) {
      const double* src = a.vhat[m] + static_cast<int64_t>(g.tco[m]) * VHS;
      for (int e = 2 * tid; e < VHS; e += 2 * THREADS) cp_async16(vh + (m - 1) * VHS + e, src + e, 16);
    }
    cp_async_commit();
    // diagonal blocks: S (0), A_m (m), Tc (D), identity/zero padded to 8x8
    for (int e = tid; e < (D + 1) * 64; e += THREADS) {
      const int b = e >> 6, r = (e >> 3) & 7, c = e & 7;
      const int m = b == D ? 0 : b;
      const double* M = b == D ? a.Tc : a.T[m];
      const int em = g.ext[m], st = g.start[m], nm = a.dims[m];
      double v;
      if (r < em && c < em) v = M[(st + r) + static_cast<int64_t>(st + c) * nm];
      else v = (r == c && b != D) ? 1.0 : 0.0;
      blk[b][8 * r + c] = v;
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- left-looking updates (distinct destinations per mode: no barrier
    //      between modes), far then near ----
    int64_t muls[D];
    {
      int64_t mul = 1;
#pragma unroll
      for (int m = 0; m < D; ++m) {
        muls[m] = mul;
        mul *= a.ntiles_mode[m];
      }
    }
#ifndef GSYD_ONEPASS
#define GSYD_ONEPASS 1
#endif
    constexpr int NPART = GSYD_ONEPASS ? 1 : 2;
    for (int part = 0; part < NPART && !(a.dbg & 4); ++part) {
      if (tid < D) {  // one thread per mode: the D flag round trips overlap
        const int d0 = (part == 0 && !GSYD_ONEPASS) ? 2 : 1, m = tid;
        if (g.tco[m] + d0 < a.ntiles_mode[m]) waitg(a, g.lt + d0 * muls[m]);
      }
      __syncthreads();
#pragma unroll 1
      for (int m = 0; m < D; ++m) {
        const int tm = g.tco[m], p = a.ntiles_mode[m];
        int klo, khi;
        if (GSYD_ONEPASS) {
          klo = tm + 1 < p ? a.bnd[m][tm + 1] : 0;
          khi = tm + 1 < p ? a.dims[m] : 0;
        } else if (part == 0) {
          klo = tm + 2 < p ? a.bnd[m][tm + 2] : 0;
          khi = tm + 2 < p ? a.dims[m] : 0;
        } else {
          klo = tm + 1 < p ? a.bnd[m][tm + 1] : 0;
          khi = tm + 1 < p ? (tm + 2 < p ? a.bnd[m][tm + 2] : a.dims[m]) : 0;
        }
        if (khi <= klo) continue;
        if (m == 0) {
          update_src<D>(a, g, xr, goff, -1.0, ep, 0, klo, khi, a.T[0], a.X);
          update_src<D>(a, g, xr, goff, -1.0, ep, 0, klo, khi, a.Tc, a.W[1]);
        } else {
          update_src<D>(a, g, lb[m - 1], goff, 1.0, ep, m, klo, khi, a.T[m], m == D - 1 ? a.X : a.W[m + 1]);
        }
      }
      __syncthreads();
    }

    // ---- R = A_1 (A_2 (... L_{d-1}) + L_2) + L_1; rhs -= Tc_tt R ----
#pragma unroll 1
    for (int m = D - 2; m >= 1; --m) {  // the first step reads L_{d-1} in place
      rmode<D>(a, g, rb, lb[m - 1], blk[m], ep, m, 1.0, m == D - 2 ? lb[D - 2] : nullptr);
      __syncthreads();
    }
    rmode<D>(a, g, rb, xr, blk[D], ep, 0, -1.0);  // rb = xr - Tc_tt R
    __syncthreads();

    // ---- base case: tail eigenbasis, mode-0 pencil back substitution ----
    // works on rb (= B~ - Tc_tt R) and xi (zeroed by the gather) in place
#pragma unroll 1
    for (int m = 1; m < D; ++m) {
      cmode<D>(a, g, rb, xi, vh + (m - 1) * VHS, ep, m);
      __syncthreads();
    }
    bool sing = false;
    {
      const int lp0 = a.tlog[0];
      for (int f = tid; f < (ep >> lp0); f += THREADS) {  // fibres along mode 0
        const int lt0 = f << lp0;
        // z = prod_m lambda_m(j_m) over the tail coordinates of the fibre
        double zr = 1.0, zi = 0.0;
        bool valid = true;
#pragma unroll
        for (int m = 1; m < D; ++m) {
          const int jm = (lt0 >> a.tsh[m]) & ((1 << a.tlog[m]) - 1);
          valid &= jm < g.ext[m];
          const double lr = vh[(m - 1) * VHS + 256 + jm], li = vh[(m - 1) * VHS + 264 + jm];
          const double nr = zr * lr - zi * li;
          zi = zr * li + zi * lr;
          zr = nr;
        }
        double br[8], bi[8];
        const int e0 = g.ext[0];
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (r < e0) {
            br[r] = rb[lt0 + r];
            bi[r] = xi[lt0 + r];
          }
        // back substitution over the Schur cells of S (last row first; all
        // indices compile-time so the fibre stays in registers);
        // M = S_tt + z Tc_tt, rk[i]: 0 1x1 cell, 1/2 first/second row of a 2x2
#pragma unroll
        for (int i = 7; i >= 0; --i) {
          if (i >= e0 || g.rk[i] == 2) continue;
          const bool two = g.rk[i] == 1 && i < 7;
          const int j = two ? i + 1 : i;
#pragma unroll
          for (int k = i + 1; k < 8; ++k) {
            if (k >= e0 || (two && k == i + 1)) continue;
            const double mr = blk[0][8 * i + k] + zr * blk[D][8 * i + k], mi = zi * blk[D][8 * i + k];
            br[i] -= mr * br[k] - mi * bi[k];
            bi[i] -= mr * bi[k] + mi * br[k];
            if (two) {
              const double nr = blk[0][8 * j + k] + zr * blk[D][8 * j + k], ni = zi * blk[D][8 * j + k];
              br[j] -= nr * br[k] - ni * bi[k];
              bi[j] -= nr * bi[k] + ni * br[k];
            }
          }
          if (!two) {
            const double mr = blk[0][9 * i] + zr * blk[D][9 * i], mi = zi * blk[D][9 * i];
            const double den = mr * mr + mi * mi;
            if (!(den > a.tiny * a.tiny)) {
              if (valid) sing = true;
              br[i] = bi[i] = 0.0;
            } else {
              const double nr = (br[i] * mr + bi[i] * mi) / den;
              bi[i] = (bi[i] * mr - br[i] * mi) / den;
              br[i] = nr;
            }
          } else {
            // [a b; c d] x = y (complex)
            const double ar = blk[0][8 * i + i] + zr * blk[D][8 * i + i], ai = zi * blk[D][8 * i + i];
            const double b_r = blk[0][8 * i + j] + zr * blk[D][8 * i + j], b_i = zi * blk[D][8 * i + j];
            const double cr = blk[0][8 * j + i] + zr * blk[D][8 * j + i], ci = zi * blk[D][8 * j + i];
            const double dr = blk[0][8 * j + j] + zr * blk[D][8 * j + j], di = zi * blk[D][8 * j + j];
            const double detr = (ar * dr - ai * di) - (b_r * cr - b_i * ci);
            const double deti = (ar * di + ai * dr) - (b_r * ci + b_i * cr);
            const double den = detr * detr + deti * deti;
            if (!(den > a.tiny * a.tiny * a.tiny * a.tiny)) {
              if (valid) sing = true;
              br[i] = bi[i] = br[j] = bi[j] = 0.0;
            } else {
              const double yir = br[i], yii = bi[i], yjr = br[j], yji = bi[j];
              const double nir = (dr * yir - di * yii) - (b_r * yjr - b_i * yji);
              const double nii = (dr * yii + di * yir) - (b_r * yji + b_i * yjr);
              const double njr = (ar * yjr - ai * yji) - (cr * yir - ci * yii);
              const double nji = (ar * yji + ai * yjr) - (cr * yii + ci * yir);
              br[i] = (nir * detr + nii * deti) / den;
              bi[i] = (nii * detr - nir * deti) / den;
              br[j] = (njr * detr + nji * deti) / den;
              bi[j] = (nji * detr - njr * deti) / den;
            }
          }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (r < e0) {
            rb[lt0 + r] = br[r];
            xi[lt0 + r] = bi[r];
          }
      }
    }
    if (sing) atomicMin(a.status, static_cast<int>(g.lt < 0x7f7f7f7e ? g.lt : 0x7f7f7f7e));
    __syncthreads();
#pragma unroll 1
    for (int m = 1; m < D; ++m) {
      cmode<D>(a, g, rb, xi, vh + (m - 1) * VHS + 128, ep, m);
      __syncthreads();
    }

    // ---- W chain: W_{d-1} = A_{d-1} X + L_{d-1}, W_m = A_m W_{m+1} + L_m ----
    // in place in the chain buffers: lb[m-1] = L_m + A_m W_{m+1}, W_d = X (rb)
#pragma unroll 1
    for (int m = D - 1; m >= 1; --m) {
      rmode<D>(a, g, lb[m - 1], lb[m - 1], blk[m], ep, m, 1.0, m == D - 1 ? rb : lb[m]);
      __syncthreads();
    }

    // ---- scatter X_t and W_m(t), release ----
    for (int l = tid; l < ep; l += THREADS) {
      const int64_t off = goff[l];
      if (off >= 0) {
        a.X[off] = rb[l];
#pragma unroll
        for (int m = 1; m < D; ++m) a.W[m][off] = lb[m - 1][l];
      }
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(a.flags + g.lt, a.epoch);
    }
  }
}

template <int D>
cudaError_t launch_g(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info) {
  auto k = solve_gsyd_kernel<D>;
  int nsm = 0, occ = 0;
  if (cudaError_t e = kernel_setup(k, 0, THREADS, &nsm, &occ); e != cudaSuccess) return e;
  int64_t grid = static_cast<int64_t>(nsm) * occ;
  if (grid > a.ntiles) grid = a.ntiles;
  if (info) *info = SolveLaunchInfo{static_cast<int>(grid), THREADS, 0, occ};
  k<<<static_cast<unsigned>(grid), THREADS, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

TileCaps solve_gsyd_caps() { return TileCaps{8, EP, EP / 2}; }

cudaError_t launch_solve_gsyd(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info) {
  if (a.ntiles <= 0) return cudaSuccess;
  switch (a.d) {
    case 3:
      return launch_g<3>(a, st, info);
    case 4:
      return launch_g<4>(a, st, info);
    case 5:
      return launch_g<5>(a, st, info);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace tsg
