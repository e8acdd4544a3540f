// Order-3 Laplace fast path: the dataflow solve specialised for d = 3 with a
// compile-time padded 16x16x16 tile (C1, C2, C4 of BASELINE.json).
//
// Per tile (one 256-thread CTA, two CTAs per SM):
//   1. host-packed tile coordinates -> per-mode tables (start, extent, Schur
//      cells, row->cell maps) in one round trip; B~_t, the three diagonal
//      blocks T_m[t,t] and the eigenbasis data are fetched with cp.async
//      (padding rows zero-filled), so all index math is shifts and masks;
//   2. left-looking updates  acc -= T_m[t, later] x_m X(later)  on DMMA with
//      fragments loaded straight from L2 (each B element feeds exactly one
//      8-row DMMA block, so shared-memory staging would buy nothing): the far
//      tiles of all modes first (released >= 2 hyperplanes ago), then the
//      three nearest neighbours;
//   3. the tile moves into the eigenbasis of its diagonal Schur blocks
//      (block-diagonal P_m^{-1} per mode, see solve_lap.cu), where the base
//      cells decouple and the wavefront over cell hyperplanes solves every
//      unknown independently (complex), then back with P_m;
//   4. scatter X_t and release its flag.
// Reference: lap_rec / lap_base (laplace.hpp:99-153), block_back_substitution
// (kernels.hpp:179-261), mode_multiply update (laplace.hpp:147).
#include <climits>
#include <cstdlib>
#include <cstring>
#include <cstdint>

#include "common.cuh"
#include "solve.h"
#include "solve_common.cuh"
#include "util.h"

namespace tsg {
namespace {

// LT = log2 of the padded tile extent: 3 (8^3 tiles, 128 threads) or
// 4 (16^3 tiles, 256 threads).
#ifndef L3_T3
#define L3_T3 128
#endif
#ifndef L3_MINB
#define L3_MINB 4
#endif
template <int LT>
struct L3C {
  static constexpr int E = 1 << LT;
  static constexpr int T = E * E * E;
  static constexpr int THREADS = LT == 3 ? L3_T3 : 256;
  static constexpr int WARPS = THREADS / 32;
  static constexpr int MB = E / 8;               // 8-row DMMA blocks along the mode
  static constexpr int NBW = E * E / 8 / WARPS;  // 8-col DMMA blocks per warp
  // shared memory layout (doubles)
  static constexpr int OFF_XR = 0;
  static constexpr int OFF_XI = OFF_XR + T;
  // per mode: That_m (re, im: E x E each) then lambda_m (re, im: E each),
  // host-precomputed per tile index (tsg_plan: dhat tables)
  static constexpr int DHS = 2 * E * E + 2 * E;
  static constexpr int OFF_DH = OFF_XI + T;
  static constexpr int OFF_PD = OFF_DH + 3 * DHS;        // eigenbasis rows: 3 x E x kPStride
  static constexpr int OFF_LAM = OFF_PD + 3 * E * kPStride;
  static_assert(LT != 3 || 3 * kVhStride <= OFF_LAM - OFF_DH, "vh aliases dh + pd");
  // K-split updates (LT = 3): every warp accumulates its partial tile
  // products in a private buffer (reused as the complex work tile of the
  // diagonalised solve)
  static constexpr bool KSPLIT = LT == 3;
  static constexpr int OFF_RED = OFF_LAM;
  static constexpr int DOUBLES = OFF_RED + (KSPLIT ? WARPS * T : 0);
  static constexpr int BYTES = DOUBLES * 8;
};

struct L3Geom {
  int64_t lt;
  int64_t gbase;
  int start[3], ext[3], tco[3];
  int nc[3], H, kp, diag, own;
  double* xb;  // (virtual) base of the slab holding the tile
  float vc[3];
  unsigned char cs[3][16], cz[3][16], cellof[3][16], cend[3][16], cplx[3][16], ckind[3][16];
  int npair[3];
  int nlane;
  unsigned short lane[2 * 16 * 16];  // representative lanes: i0 | i1 << 4 | b2 << 8
  // mode-2 data per (cell c2, row bit b): i2 | cend << 5 | ckind << 10 | sigma << 12 | valid << 17
  unsigned m2[16][2];
  double m2lam[16][2][2];
  unsigned char prow[3][8];  // first rows of the 2x2 blocks per mode
};

// tile-local padded offset of (i0, i1, i2)
template <int LT>
TSG_DEVINL int l3off(int i0, int i1, int i2) { return i0 | (i1 << LT) | (i2 << (2 * LT)); }

// ---- left-looking update along mode M over global rows [k_lo, k_hi) --------
// xr[row i of mode M, cross-section n] -= sum_k T_M[start+i, k] X(..k..)
// Warp w owns cross-section columns [32w, 32w+32) (4 DMMA col blocks) and
// both 8-row blocks.  Fragments come straight from global memory (L2).
template <int LT, int M>
TSG_DEVINL void l3_update(const SolveArgs& a, const L3Geom& tg, double* xr, int k_lo, int k_hi) {
  using C = L3C<LT>;
  constexpr int E = C::E, MB = C::MB, NBW = C::NBW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  constexpr int VA = (M == 0) ? 1 : 0, VB = (M == 2) ? 1 : 2;  // the other two modes
  const int nm = a.dims[M];
  const double* __restrict__ Tm = a.T[M];
  const double* __restrict__ X = a.X;
  const int64_t sM = a.stride[M];
  // B fragment columns of this lane: n = 8*NBW*warp + 8*jb + gq;
  // cross-section n = ia + E*ib over modes (VA, VB).
  int64_t boff[NBW];
  bool bok[NBW];
#pragma unroll
  for (int jb = 0; jb < NBW; ++jb) {
    const int n = 8 * NBW * warp + 8 * jb + gq;
    const int ia = n & (E - 1), ib = n >> LT;
    bok[jb] = ia < tg.ext[VA] && ib < tg.ext[VB];
    boff[jb] = bok[jb] ? static_cast<int64_t>(tg.start[VA] + ia) * a.stride[VA] +
                             static_cast<int64_t>(tg.start[VB] + ib) * a.stride[VB]
                       : 0;
  }
  const int row0 = tg.start[M];
  const int em = tg.ext[M];
  {
    // a DMMA column block is fully padded when its slowest cross-section
    // index lies beyond the tile (warp-uniform): skip the warp entirely
    bool any = false;
#pragma unroll
    for (int jb = 0; jb < NBW; ++jb) any |= ((8 * NBW * warp + 8 * jb) >> LT) < tg.ext[VB];
    if (!any && !(a.dbg & 128)) return;
  }
  bool aok[MB];
#pragma unroll
  for (int ib = 0; ib < MB; ++ib) aok[ib] = gq + 8 * ib < em;
  double c[MB][NBW][2];
#pragma unroll
  for (int ib = 0; ib < MB; ++ib)
#pragma unroll
    for (int jb = 0; jb < NBW; ++jb) c[ib][jb][0] = c[ib][jb][1] = 0.0;

  // Per-lane pointers at row k_lo + tq.  Padded rows/columns read in-bounds
  // garbage that only reaches padded outputs (never scattered); only the
  // K tail is masked.
  const double* pa[MB];
  const double* pb[NBW];
#pragma unroll
  for (int ib = 0; ib < MB; ++ib) {
    const int row = aok[ib] ? row0 + gq + 8 * ib : row0;
    pa[ib] = Tm + static_cast<int64_t>(k_lo + tq) * nm + row;
  }
#pragma unroll
  for (int jb = 0; jb < NBW; ++jb) pb[jb] = X + boff[jb] + static_cast<int64_t>(k_lo + tq) * sM;
  const int64_t sa = 4 * static_cast<int64_t>(nm), sb = 4 * sM;
  constexpr int U = 4;  // k4-steps per batch (16 rows)
  const int kr = k_hi - k_lo;
  const int nfull = kr >> 4;
  for (int bt = 0; bt < nfull; ++bt) {
    double af[U][MB], bf[U][NBW];
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int ib = 0; ib < MB; ++ib) {
        af[u][ib] = __ldg(pa[ib]);
        pa[ib] += sa;
      }
#pragma unroll
      for (int jb = 0; jb < NBW; ++jb) {
        bf[u][jb] = ld_cg(pb[jb]);
        pb[jb] += sb;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int ib = 0; ib < MB; ++ib)
#pragma unroll
        for (int jb = 0; jb < NBW; ++jb) dmma(c[ib][jb][0], c[ib][jb][1], af[u][ib], bf[u][jb]);
  }
  const int rem = kr & 15;
  if (rem) {
    double af[U][MB], bf[U][NBW];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool kok = 4 * u + tq < rem;
#pragma unroll
      for (int ib = 0; ib < MB; ++ib) {
        af[u][ib] = kok ? __ldg(pa[ib]) : 0.0;
        pa[ib] += sa;
      }
#pragma unroll
      for (int jb = 0; jb < NBW; ++jb) {
        bf[u][jb] = kok ? ld_cg(pb[jb]) : 0.0;
        pb[jb] += sb;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (4 * u >= rem) break;
#pragma unroll
      for (int ib = 0; ib < MB; ++ib)
#pragma unroll
        for (int jb = 0; jb < NBW; ++jb) dmma(c[ib][jb][0], c[ib][jb][1], af[u][ib], bf[u][jb]);
    }
  }
  // xr -= c   (rows i = 8*ib + gq, cols n = 8*NBW*warp + 8*jb + 2*tq + h)
#pragma unroll
  for (int ib = 0; ib < MB; ++ib)
#pragma unroll
    for (int jb = 0; jb < NBW; ++jb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = 8 * ib + gq, n = 8 * NBW * warp + 8 * jb + 2 * tq + h;
        const int ia = n & (E - 1), ib2 = n >> LT;
        int l;
        if (M == 0) l = l3off<LT>(i, ia, ib2);
        else if (M == 1) l = l3off<LT>(ia, i, ib2);
        else l = l3off<LT>(ia, ib2, i);
        xr[l] -= c[ib][jb][h];
      }
}

// slab (owner) of row `row` along the last mode
TSG_DEVINL int slab_of(const SolveArgs& a, int row) {
  int q = 0;
  while (q + 1 < a.nslab && row >= a.slo[q + 1]) ++q;
  return q;
}

TSG_DEVINL void wait_flag(const SolveArgs& a, int64_t tile, int owner, int own) {
  if (a.dbg & 512) return;  // timing ablation only: results are wrong
  const int* f = a.fs[owner] + tile;
  unsigned ns = 32;
  const unsigned cap = (a.dbg & 64) ? 32 : 256;
  if (a.sys && owner != own) {  // released by a peer GPU
    while (ld_acquire_sys(f) < a.epoch) {
      __nanosleep(ns);
      if (ns < cap) ns <<= 1;
    }
    return;
  }
  while (ld_acquire(f) < a.epoch) {
    __nanosleep(ns);
    if (ns < cap) ns <<= 1;
  }
}

// single-tensor (one GPU, one slab) flag wait
TSG_DEVINL void wait_flag1(const SolveArgs& a, int64_t tile) {
  if (a.dbg & 512) return;  // timing ablation only: results are wrong
  const int* f = a.flags + tile;
  unsigned ns = 32;
  const unsigned cap = (a.dbg & 64) ? 32 : 256;
  while (ld_acquire(f) < a.epoch) {
    __nanosleep(ns);
    if (ns < cap) ns <<= 1;
  }
}

// ---- far updates of all three modes in one pass, K split across warps ------
// The k4-steps of the three far ranges (rows >= bnd[t_m + 3] of each mode)
// are concatenated and cut into WARPS equal slices.  A warp accumulates the
// whole E x E^2 product of its current mode in registers (one 8-row block,
// all E column blocks) and, at a mode change or the end of its slice, folds
// it into xr (warp 0, subtracting) or its private buffer (adding; folded
// into xr after the near updates).  Every warp thus walks a quarter of the
// K range instead of all of it: 4x fewer dependent L2 round trips per tile
// than splitting the columns.
#ifndef L3_PARWAIT
#define L3_PARWAIT 1
#endif
#ifndef L3_UB
#define L3_UB 2
#endif
template <int LT, int M, bool VOL>
TSG_DEVINL void l3_far_seg(const SolveArgs& a, const L3Geom& tg, const double* xb, int k_lo, int k_hi,
                           double* dst, bool sub) {
  constexpr int E = L3C<LT>::E, UB = L3_UB;
  static_assert(E == 8, "one 8-row DMMA block per mode");
  const int lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  constexpr int VA = (M == 0) ? 1 : 0, VB = (M == 2) ? 1 : 2;  // the other two modes
  const int nm = a.dims[M];
  const int ea = tg.ext[VA], eb = tg.ext[VB], em = tg.ext[M];
  // B column n = 8 jb + gq  <->  cross-section (VA = gq, VB = jb)
  const int64_t SJ = a.stride[VB];
  const int ia = gq < ea ? gq : ea - 1;  // padded lanes re-read a valid column
  const int64_t base = static_cast<int64_t>(tg.start[VA] + ia) * a.stride[VA] +
                       static_cast<int64_t>(tg.start[VB]) * SJ;
  const int row = tg.start[M] + (gq < em ? gq : em - 1);
  const double* pa = a.T[M] + static_cast<int64_t>(k_lo + tq) * nm + row;
  const double* pb = xb + base + static_cast<int64_t>(k_lo + tq) * a.stride[M];
  const int64_t sa = 4 * static_cast<int64_t>(nm), sb = 4 * a.stride[M];
  double c[E][2];
#pragma unroll
  for (int jb = 0; jb < E; ++jb) c[jb][0] = c[jb][1] = 0.0;
  const int nfs = (k_hi - k_lo) >> 2;  // k4-steps with all four rows valid
  const int nb = nfs / UB;
  for (int bt = 0; bt < nb; ++bt) {
    double af[UB], bf[UB][E];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      af[u] = __ldg(pa);
      pa += sa;
#pragma unroll
      for (int jb = 0; jb < E; ++jb) bf[u][jb] = jb < eb ? (VOL ? ld_volatile(pb + jb * SJ) : ld_cg(pb + jb * SJ)) : 0.0;
      pb += sb;
    }
#pragma unroll
    for (int u = 0; u < UB; ++u)
#pragma unroll
      for (int jb = 0; jb < E; ++jb)
        if (jb < eb) dmma(c[jb][0], c[jb][1], af[u], bf[u][jb]);
  }
  // remaining steps (the last one possibly partial), masked per row
  for (int k = k_lo + 4 * nb * UB; k < k_hi; k += 4) {
    const bool kok = k + tq < k_hi;
    const double av = kok ? __ldg(pa) : 0.0;
    double bv[E];
#pragma unroll
    for (int jb = 0; jb < E; ++jb)
      bv[jb] = (kok && jb < eb) ? (VOL ? ld_volatile(pb + jb * SJ) : ld_cg(pb + jb * SJ)) : 0.0;
    pa += sa;
    pb += sb;
#pragma unroll
    for (int jb = 0; jb < E; ++jb)
      if (jb < eb) dmma(c[jb][0], c[jb][1], av, bv[jb]);
  }
  // fold: row i = gq of mode M, cross-section (VA = 2 tq + h, VB = jb)
#pragma unroll
  for (int jb = 0; jb < E; ++jb)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = gq, va = 2 * tq + h;
      int l;
      if (M == 0) l = l3off<LT>(i, va, jb);
      else if (M == 1) l = l3off<LT>(va, i, jb);
      else l = l3off<LT>(va, jb, i);
      dst[l] += sub ? -c[jb][h] : c[jb][h];
    }
}

// Single-tensor variant: one K range per mode (rows [klo_m, khi_m)), the
// mode loop unrolled at compile time.
template <int LT>
TSG_DEVINL void l3_ksplit1(const SolveArgs& a, const L3Geom& tg, double* red, const int* klo,
                           const int* khi) {
  using C = L3C<LT>;
  const int warp = threadIdx.x >> 5;
  int s[3], S = 0;
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    s[m] = (khi[m] - klo[m] + 3) >> 2;
    S += s[m];
  }
  if (S == 0) return;
  const int w0 = (S * warp) / C::WARPS, w1 = (S * (warp + 1)) / C::WARPS;
  double* dst = red + warp * C::T;
  int off = 0;
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    const int lo = w0 > off ? w0 : off, hi = w1 < off + s[m] ? w1 : off + s[m];
    if (lo < hi) {
      const int kl = klo[m] + 4 * (lo - off);
      const int kh = min(khi[m], klo[m] + 4 * (hi - off));
      if (m == 0) l3_far_seg<LT, 0, false>(a, tg, a.X, kl, kh, dst, false);
      else if (m == 1) l3_far_seg<LT, 1, false>(a, tg, a.X, kl, kh, dst, false);
      else l3_far_seg<LT, 2, false>(a, tg, a.X, kl, kh, dst, false);
    }
    off += s[m];
  }
}

// One K range of the updates: rows [k_lo, k_hi) of mode m, read through the
// (virtual) base of the slab that holds them.
struct KSeg {
  int m, k_lo, k_hi, remote;
  const double* xb;
};

template <int LT>
TSG_DEVINL void l3_far_ksplit(const SolveArgs& a, const L3Geom& tg, double* red, const KSeg* seg,
                              int nseg) {
  using C = L3C<LT>;
  const int warp = threadIdx.x >> 5;
  int S = 0;
  for (int i = 0; i < nseg; ++i) S += (seg[i].k_hi - seg[i].k_lo + 3) >> 2;
  if (S == 0) return;
  const int w0 = (S * warp) / C::WARPS, w1 = (S * (warp + 1)) / C::WARPS;
  double* dst = red + warp * C::T;
  int off = 0;
  for (int i = 0; i < nseg; ++i) {
    const int si = (seg[i].k_hi - seg[i].k_lo + 3) >> 2;
    const int lo = w0 > off ? w0 : off, hi = w1 < off + si ? w1 : off + si;
    if (lo < hi) {
      const int kl = seg[i].k_lo + 4 * (lo - off);
      const int kh = min(seg[i].k_hi, seg[i].k_lo + 4 * (hi - off));
      const double* xb = seg[i].xb;
      if (seg[i].m == 0) l3_far_seg<LT, 0, false>(a, tg, xb, kl, kh, dst, false);
      else if (seg[i].m == 1) l3_far_seg<LT, 1, false>(a, tg, xb, kl, kh, dst, false);
      else if (seg[i].remote) l3_far_seg<LT, 2, true>(a, tg, xb, kl, kh, dst, false);
      else l3_far_seg<LT, 2, false>(a, tg, xb, kl, kh, dst, false);
    }
    off += si;
  }
}

// Update segments for rows [lo_m, hi_m) of each mode: modes 0, 1 read the
// tile's own slab; mode 2 is cut at slab boundaries.
TSG_DEVINL int l3_segments(const SolveArgs& a, int own, const int* lo, const int* hi, KSeg* seg) {
  int n = 0;
  for (int m = 0; m < 2; ++m)
    if (hi[m] > lo[m]) seg[n++] = KSeg{m, lo[m], hi[m], 0, a.xs[own]};
  if (hi[2] > lo[2]) {
    for (int q = slab_of(a, lo[2]); q < a.nslab && a.slo[q] < hi[2]; ++q) {
      const int kl = max(lo[2], a.slo[q]), kh = min(hi[2], a.slo[q + 1]);
      if (kh > kl) seg[n++] = KSeg{2, kl, kh, (a.sys && q != own) ? 1 : 0, a.xs[q]};
    }
  }
  return n;
}

// ---- diagonalised tiles ------------------------------------------------------
// When the eigenvector bases V_m of the tile's three diagonal blocks are well
// conditioned (host vcond tables), the in-tile Kronecker-sum solve is
//   x^ = x x_0 V0^-1 x_1 V1^-1 x_2 V2^-1,  x^ /= l0_i + l1_j + l2_k,
//   x  = x^ x_0 V0 x_1 V1 x_2 V2
// i.e. six complex 8x8 mode products on DMMA (real input for the first, real
// output for the last) and no wavefront.  Warp w owns cross-section column
// blocks 2w and 2w+1; the matrix is row-major (8 x 8) in shared memory.
template <int M>
TSG_DEVINL int l3d_addr(int i, int n) {  // tile offset of mode-M row i, cross-section column n
  if (M == 0) return i + 8 * n;
  if (M == 1) return (n & 7) + 8 * i + 64 * (n >> 3);
  return n + 64 * i;
}

template <int M, bool CIN, bool COUT, bool DIV>
TSG_DEVINL bool l3d_mode(const double* sr, const double* si, double* dr, double* di, const double* Ar,
                         const double* Ai, const double* vh, const int* ext, double tiny) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double cr[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, ci[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    const int k = 4 * ks + t;
    const double ar = Ar[8 * g + k], ai = Ai[8 * g + k];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int n = 8 * (2 * warp + q) + g;
      const double br = sr[l3d_addr<M>(k, n)];
      dmma(cr[q][0], cr[q][1], ar, br);
      if (COUT) dmma(ci[q][0], ci[q][1], ai, br);
      if (CIN) {
        const double bi = si[l3d_addr<M>(k, n)];
        dmma(cr[q][0], cr[q][1], -ai, bi);
        if (COUT) dmma(ci[q][0], ci[q][1], ar, bi);
      }
    }
  }
  bool sing = false;
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = 8 * (2 * warp + q) + 2 * t + h;
      double vr = cr[q][h], vi = ci[q][h];
      if (DIV) {  // M == 2: rows are i2, columns (i0, i1)
        const int i0 = n & 7, i1 = n >> 3;
        const double mr = vh[4 * 64 + i0] + vh[kVhStride + 4 * 64 + i1] + vh[2 * kVhStride + 4 * 64 + g];
        const double mi = vh[4 * 64 + 8 + i0] + vh[kVhStride + 4 * 64 + 8 + i1] +
                          vh[2 * kVhStride + 4 * 64 + 8 + g];
        const double den = mr * mr + mi * mi;
        if (!(den > tiny * tiny)) {
          if (i0 < ext[0] && i1 < ext[1] && g < ext[2]) sing = true;
          vr = vi = 0.0;
        } else {
          const double inv = 1.0 / den;
          const double r = (cr[q][h] * mr + ci[q][h] * mi) * inv;
          vi = (ci[q][h] * mr - cr[q][h] * mi) * inv;
          vr = r;
        }
      }
      dr[l3d_addr<M>(g, n)] = vr;
      if (COUT) di[l3d_addr<M>(g, n)] = vi;
    }
  return sing;
}

// DIST = the tensor is split into slabs (multi-GPU or emulated, tsg_dplan):
// per-slab bases, owner-aware flags and segment lists; the single-tensor
// instantiation keeps the plain addressing.
template <int LT, bool DIST>
__global__ void __launch_bounds__(L3C<LT>::THREADS, LT == 3 ? L3_MINB : 2)
    solve_lap3_kernel(SolveArgs a) {
  pdl_wait();
  pdl_trigger();
  using C = L3C<LT>;
  constexpr int E = C::E, L3_T = C::T, L3_THREADS = C::THREADS;
  constexpr int EE = E * E, MSK = E - 1;
  extern __shared__ __align__(16) double smem[];
  __shared__ L3Geom tg;
  __shared__ int s_tile;
  __shared__ KSeg s_seg[2][2 + kMaxSlabs];  // far / near pass segments (DIST)
  __shared__ int s_nseg[2];
  double* xr = smem + C::OFF_XR;
  double* xi = smem + C::OFF_XI;
  double* dh = smem + C::OFF_DH;
  double* pd = smem + C::OFF_PD;
  double* lam = smem + C::OFF_LAM;
  double* red = smem + C::OFF_RED;
  const int tid = threadIdx.x;
  unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tmark = clock64();
  auto mark = [&](int k) {
    if (a.prof) {
      const long long t = clock64();
      ph[k] += static_cast<unsigned long long>(t - tmark);
      tmark = t;
    }
  };

  for (;;) {
    mark(7);
    if (tid == 0) s_tile = atomicAdd(a.counter, 1);
    __syncthreads();
    const int qi = s_tile;
    if (qi >= a.ntiles) break;
    mark(0);

    // ---- geometry (host-built tables) ---------------------------------------
    if (tid < 3) {
      const unsigned long long pk = a.ocoord[qi];
      const int tm = static_cast<int>((pk >> (10 * tid)) & 1023);
      const TileMode& src = a.tmode[tid][tm];
      tg.tco[tid] = tm;
      tg.start[tid] = src.start;
      tg.ext[tid] = src.ext;
      tg.nc[tid] = src.nc;
      tg.vc[tid] = src.vcond;
      for (int k = 0; k < 16; ++k) {
        tg.cs[tid][k] = src.cs[k];
        tg.cz[tid][k] = src.cz[k];
        tg.cellof[tid][k] = src.cellof[k];
        tg.cend[tid][k] = src.cend[k];
        tg.cplx[tid][k] = src.cplx[k];
        tg.ckind[tid][k] = src.ckind[k];
      }
      if (tid == 0) tg.lt = a.order[qi];
    }
    __syncthreads();
    if (tid == 0) {
      if constexpr (DIST) {
        tg.own = slab_of(a, tg.start[2]);
        tg.xb = a.xs[tg.own];
      }
      tg.gbase = static_cast<int64_t>(tg.start[0]) * a.stride[0] +
                 static_cast<int64_t>(tg.start[1]) * a.stride[1] +
                 static_cast<int64_t>(tg.start[2]) * a.stride[2];
      tg.H = tg.nc[0] + tg.nc[1] + tg.nc[2] - 3;
      int kp = 0;
      for (int m = 0; m < 3; ++m) {
        int np = 0;
        for (int k = 0; k < tg.nc[m]; ++k)
          if (tg.cz[m][k] == 2) tg.prow[m][np++] = tg.cs[m][k];
        tg.npair[m] = np;
        kp |= np ? (1 << m) : 0;
      }
      tg.kp = kp;
      tg.diag = LT == 3 && a.vhat[0] != nullptr && !(a.dbg & 1024) &&
                tg.vc[0] * tg.vc[1] * tg.vc[2] <= kDiagCond;
    }
    __syncthreads();
    const int e0 = tg.ext[0], e1 = tg.ext[1], e2 = tg.ext[2];

    // ---- gather B~_t (padded, zero-filled) + diag blocks + eigenbasis rows ----
    for (int l = tid; l < L3_T; l += L3_THREADS) {
      const int i0 = l & MSK, i1 = (l >> LT) & MSK, i2 = l >> (2 * LT);
      const bool ok = i0 < e0 && i1 < e1 && i2 < e2;
      const double* xb = DIST ? tg.xb : a.X;
      const double* src = ok ? xb + tg.gbase + i0 + i1 * a.stride[1] + i2 * a.stride[2] : a.X;
      cp_async8(xr + l, src, ok ? 8 : 0);
    }
    if (tg.diag) {  // eigenvector bases (V^-1, V, lambda) of the three modes
      double* vh = dh;  // aliases the That / eigenbasis-row regions
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const double* vsrc = a.vhat[m] + static_cast<int64_t>(tg.tco[m]) * kVhStride;
        for (int e = 2 * tid; e < kVhStride; e += 2 * L3_THREADS)
          cp_async16(vh + m * kVhStride + e, vsrc + e, 16);
      }
    } else {
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int em = tg.ext[m], st = tg.start[m];
        const double* dsrc = a.dhat[m] + static_cast<int64_t>(tg.tco[m]) * C::DHS;
        for (int e = 2 * tid; e < C::DHS; e += 2 * L3_THREADS)
          cp_async16(dh + m * C::DHS + e, dsrc + e, 16);
        for (int e = tid; e < E * kPStride; e += L3_THREADS) {
          const bool ok = e < em * kPStride;
          cp_async8(pd + m * E * kPStride + e,
                    ok ? a.pdat[m] + static_cast<int64_t>(st) * kPStride + e : a.pdat[m], ok ? 8 : 0);
        }
      }
    }
    cp_async_commit();

    // ---- left-looking updates ---------------------------------------------------
    int64_t mul[3] = {1, a.ntiles_mode[0], static_cast<int64_t>(a.ntiles_mode[0]) * a.ntiles_mode[1]};
    if constexpr (C::KSPLIT) {
      // Two K-split passes over all three modes, each one batch of DMMA
      // fragment loads per warp and slice (see l3_far_ksplit); the staged
      // copies land meanwhile (the passes only read global memory and fold
      // into the per-warp buffers):
      //   far  = rows of tiles >= t+3 (released >= 3 hyperplanes ago),
      //   near = rows of tiles t+1, t+2 (after the t+1 flags).
      {
        double* mine = red + (tid >> 5) * L3_T;
        for (int l = tid & 31; l < L3_T; l += 32) mine[l] = 0.0;
        __syncwarp();
      }
      if constexpr (!DIST) {
        int klo[3], khi[3];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          const int tm = tg.tco[m];
          const bool has = tm + 3 < a.ntiles_mode[m] && !(a.dbg & 4);
          klo[m] = has ? a.bnd[m][tm + 3] : 0;
          khi[m] = has ? a.dims[m] : 0;
          if (has && tid == 0) wait_flag1(a, tg.lt + 3 * mul[m]);
        }
        __syncthreads();
        mark(3);
        l3_ksplit1<LT>(a, tg, red, klo, khi);
        mark(4);
#if L3_PARWAIT
        int64_t wt[3];
#endif
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          const int tm = tg.tco[m];
          const bool has = tm + 1 < a.ntiles_mode[m] && !(a.dbg & 4);
          klo[m] = has ? a.bnd[m][tm + 1] : 0;
          khi[m] = has ? (tm + 3 < a.ntiles_mode[m] ? a.bnd[m][tm + 3] : a.dims[m]) : 0;
#if L3_PARWAIT
          wt[m] = has ? tg.lt + mul[m] : -1;
#else
          if (has && tid == 0) wait_flag1(a, tg.lt + mul[m]);
#endif
        }
#if L3_PARWAIT
        if (tid == 0 && !(a.dbg & 512)) {
          bool ok[3] = {wt[0] < 0, wt[1] < 0, wt[2] < 0};
          unsigned ns = 32;
          while (!(ok[0] && ok[1] && ok[2])) {
            int v[3];
#pragma unroll
            for (int m = 0; m < 3; ++m) v[m] = ok[m] ? 0 : ld_acquire(a.flags + wt[m]);
#pragma unroll
            for (int m = 0; m < 3; ++m) ok[m] = ok[m] || v[m] >= a.epoch;
            if (ok[0] && ok[1] && ok[2]) break;
            __nanosleep(ns);
            if (ns < 256) ns <<= 1;
          }
        }
#endif
        __syncthreads();
        mark(2);
        l3_ksplit1<LT>(a, tg, red, klo, khi);
      } else {
      if (tid == 0) {  // far: rows of tiles >= t+3
        int lo[3], hi[3];
        for (int m = 0; m < 3; ++m) {
          const int tm = tg.tco[m];
          const bool has = tm + 3 < a.ntiles_mode[m] && !(a.dbg & 4);
          lo[m] = has ? a.bnd[m][tm + 3] : 0;
          hi[m] = has ? a.dims[m] : 0;
          if (has) wait_flag(a, tg.lt + 3 * mul[m], m == 2 ? slab_of(a, lo[2]) : tg.own, tg.own);
        }
        s_nseg[0] = l3_segments(a, tg.own, lo, hi, s_seg[0]);
      }
      __syncthreads();
      mark(3);
      l3_far_ksplit<LT>(a, tg, red, s_seg[0], s_nseg[0]);
      mark(4);
      if (tid == 0) {  // near: rows of tiles t+1, t+2
        int lo[3], hi[3];
        for (int m = 0; m < 3; ++m) {
          const int tm = tg.tco[m];
          const bool has = tm + 1 < a.ntiles_mode[m] && !(a.dbg & 4);
          lo[m] = has ? a.bnd[m][tm + 1] : 0;
          hi[m] = has ? (tm + 3 < a.ntiles_mode[m] ? a.bnd[m][tm + 3] : a.dims[m]) : 0;
          if (has) wait_flag(a, tg.lt + mul[m], m == 2 ? slab_of(a, lo[2]) : tg.own, tg.own);
        }
        s_nseg[1] = l3_segments(a, tg.own, lo, hi, s_seg[1]);
      }
      __syncthreads();
      mark(2);
      l3_far_ksplit<LT>(a, tg, red, s_seg[1], s_nseg[1]);
      }
      cp_async_wait_all();
      __syncthreads();
      mark(1);
      for (int l = tid; l < L3_T; l += L3_THREADS) {
        double r = 0.0;
#pragma unroll
        for (int w = 0; w < C::WARPS; ++w) r += red[w * L3_T + l];
        xr[l] -= r;
        if (!tg.diag) xi[l] = 0.0;
      }
      __syncthreads();
    } else {
      cp_async_wait_all();
      __syncthreads();
      mark(1);
      // parts by distance along each mode, farthest first across modes:
      // part 0 = tiles >= t+3, part 1 = t+2, part 2 = t+1
      for (int part = 0; part < 3; ++part) {
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          const int tm = tg.tco[m], pmt = a.ntiles_mode[m];
          const int* bm = a.bnd[m];
          const int dist = part == 0 ? 3 : (part == 1 ? 2 : 1);
          if (tm + dist >= pmt || (a.dbg & 4)) continue;  // uniform
          const int k_lo = bm[tm + dist];
          const int k_hi = part == 0 ? a.dims[m] : bm[tm + dist + 1];
          const int64_t wtile = tg.lt + dist * mul[m];
          if (tid == 0) wait_flag1(a, wtile);
          __syncthreads();
          if (m == 0) l3_update<LT, 0>(a, tg, xr, k_lo, k_hi);
          else if (m == 1) l3_update<LT, 1>(a, tg, xr, k_lo, k_hi);
          else l3_update<LT, 2>(a, tg, xr, k_lo, k_hi);
        }
      }
      __syncthreads();
      mark(2);
      for (int l = tid; l < L3_T; l += L3_THREADS) xi[l] = 0.0;
      __syncthreads();
    }

    if constexpr (LT == 3) {
      if (tg.diag) {
        const double* vh = dh;
        double* yr = red;
        double* yi = red + L3_T;
        const int* ex = tg.ext;
        constexpr int VS = kVhStride, RE = 0, IM = 64, VR = 128, VI = 192;
        bool sing = false;
        l3d_mode<0, false, true, false>(xr, nullptr, yr, yi, vh + RE, vh + IM, vh, ex, a.tiny);
        __syncthreads();
        l3d_mode<1, true, true, false>(yr, yi, xr, xi, vh + VS + RE, vh + VS + IM, vh, ex, a.tiny);
        __syncthreads();
        sing |= l3d_mode<2, true, true, true>(xr, xi, yr, yi, vh + 2 * VS + RE, vh + 2 * VS + IM, vh, ex,
                                              a.tiny);
        __syncthreads();
        l3d_mode<2, true, true, false>(yr, yi, xr, xi, vh + 2 * VS + VR, vh + 2 * VS + VI, vh, ex, a.tiny);
        __syncthreads();
        l3d_mode<1, true, true, false>(xr, xi, yr, yi, vh + VS + VR, vh + VS + VI, vh, ex, a.tiny);
        __syncthreads();
        l3d_mode<0, true, false, false>(yr, yi, xr, nullptr, vh + VR, vh + VI, vh, ex, a.tiny);
        if (sing) atomicMin(a.status, static_cast<int>(tg.lt < 0x7f7f7f7e ? tg.lt : 0x7f7f7f7e));
        __syncthreads();
        mark(5);
        goto scatter;
      }
    }
    {
    // ---- into the eigenbasis (pair modes) -------------------------------------
    const int kp = tg.kp;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      if (!(kp & (1 << m))) continue;  // uniform
      const double* pm = pd + m * E * kPStride;
      // work item: (2x2 block of mode m, cross-section n)
      const int nw = tg.npair[m] * EE;
      for (int w = tid; w < nw; w += L3_THREADS) {
        const int i = tg.prow[m][w >> (2 * LT)], n = w & (EE - 1);
        const int na = n & MSK, nb = n >> LT;
        int l, st;
        if (m == 0) l = l3off<LT>(i, na, nb), st = 1;
        else if (m == 1) l = l3off<LT>(na, i, nb), st = E;
        else l = l3off<LT>(na, nb, i), st = EE;
        const double* pi = pm + i * kPStride + 12;
        const int l2 = l + st;
        const double ar = xr[l], ai = xi[l], br = xr[l2], bi = xi[l2];
        xr[l] = pi[0] * ar - pi[1] * ai + pi[2] * br - pi[3] * bi;
        xi[l] = pi[0] * ai + pi[1] * ar + pi[2] * bi + pi[3] * br;
        xr[l2] = pi[4] * ar - pi[5] * ai + pi[6] * br - pi[7] * bi;
        xi[l2] = pi[4] * ai + pi[5] * ar + pi[6] * bi + pi[7] * br;
      }
      __syncthreads();
    }

    mark(3);
    // ---- wavefront over cell hyperplanes --------------------------------------
    // lanes: (slot over the (c0, c1) cell grid) x (unknown inside the cell).
    // Modes 0 and 1 of a lane are fixed for the whole tile; only the mode-2
    // cell c2 = h - c0 - c1 moves with the hyperplane.
    // Conjugate symmetry: the tile data are real, so in the eigenbasis
    // xhat(sigma(u)) = conj(xhat(u)) with sigma swapping the two rows of every
    // complex-pair block (same cell, same hyperplane).  Lanes are the orbit
    // representatives (i0, i1, b2): the first complex-pair row decides; each
    // solve writes u and sigma(u).
    const int nc2 = tg.nc[2];
    const int p2 = (kp & 4) ? 1 : 0;
    if (tid == 0) tg.nlane = 0;
    __syncthreads();
    for (int L = tid; L < (EE << p2); L += L3_THREADS) {
      const int rest = L >> p2;
      const int i0 = rest & (E - 1), i1 = (rest >> LT) & (E - 1), b2 = L & p2;
      if (i0 >= tg.ext[0] || i1 >= tg.ext[1]) continue;
      const int k0 = tg.ckind[0][i0], k1 = tg.ckind[1][i1];
      if (k0 == 2 || (k0 == 0 && k1 == 2)) continue;  // represented by its partner
      tg.lane[atomicAdd(&tg.nlane, 1)] = static_cast<unsigned short>(i0 | (i1 << 4) | (b2 << 8));
    }
    __syncthreads();
    const int nlane = tg.nlane;
    constexpr int LPT = (2 * EE + L3_THREADS - 1) / L3_THREADS;  // lanes per thread
    int lc01[LPT], lb2[LPT], loff[LPT], lce0[LPT], lce1[LPT], li0[LPT], li1[LPT], lsoff[LPT];
    double llr[LPT], lli[LPT];
    bool lok[LPT], lcx[LPT];
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
      const int L = tid + q * L3_THREADS;
      lok[q] = L < nlane;
      const int pk = lok[q] ? tg.lane[L] : 0;
      const int i0 = pk & 15, i1 = (pk >> 4) & 15, b2 = (pk >> 8) & 1;
      const int k0 = tg.ckind[0][i0], k1 = tg.ckind[1][i1];
      lc01[q] = tg.cellof[0][i0] + tg.cellof[1][i1];
      lb2[q] = b2;
      li0[q] = i0;
      li1[q] = i1;
      loff[q] = i0 + E * i1;
      lcx[q] = k0 != 0 || k1 != 0;
      // sigma of the (i0, i1) part of the offset
      lsoff[q] = (k0 == 1 ? i0 + 1 : i0) + E * (k1 == 1 ? i1 + 1 : (k1 == 2 ? i1 - 1 : i1));
      lce0[q] = tg.cend[0][i0];
      lce1[q] = tg.cend[1][i1];
      llr[q] = dh[2 * EE + i0] + dh[C::DHS + 2 * EE + i1];
      lli[q] = dh[2 * EE + E + i0] + dh[C::DHS + 2 * EE + E + i1];
    }
    if (tid < 2 * nc2) {
      const int c2 = tid >> 1, b = tid & 1;
      const int r0 = tg.cs[2][c2], z = tg.cz[2][c2];
      const int i2 = r0 + (b && z == 2 ? 1 : 0);
      const int k2 = tg.ckind[2][i2];
      const int sg = k2 == 1 ? i2 + 1 : (k2 == 2 ? i2 - 1 : i2);
      const int valid = (b == 0 || z == 2) ? 1 : 0;
      tg.m2[c2][b] = static_cast<unsigned>(i2 | ((r0 + z) << 5) | (k2 << 10) | (sg << 12) | (valid << 17));
      tg.m2lam[c2][b][0] = dh[2 * C::DHS + 2 * EE + i2];
      tg.m2lam[c2][b][1] = dh[2 * C::DHS + 2 * EE + E + i2];
    }
    __syncthreads();
    bool singular = false;
    const int e0w = tg.ext[0], e1w = tg.ext[1], e2w = tg.ext[2];
    for (int h = tg.H; h >= 0; --h) {
#pragma unroll
      for (int q = 0; q < LPT; ++q) {
        const int c2 = h - lc01[q];
        if (!lok[q] || c2 < 0 || c2 >= nc2) continue;
        const unsigned pk2 = tg.m2[c2][lb2[q]];
        if (!(pk2 >> 17)) continue;
        const int i2 = pk2 & 31, ce2 = (pk2 >> 5) & 31, k2 = (pk2 >> 10) & 3, sg2 = (pk2 >> 12) & 31;
        // second row of a mode-2 complex pair: the partner lane (b2 = 0)
        // owns this orbit unless modes 0/1 already decided it
        if (lb2[q] && !lcx[q] && k2 == 2) continue;
        const int off = loff[q] + EE * i2;
        const bool orbit2 = lcx[q] || k2 != 0;  // sigma(u) != u
        const int soff = lsoff[q] + EE * sg2;
        const double mur = llr[q] + tg.m2lam[c2][lb2[q]][0];
        const double mui = lli[q] + tg.m2lam[c2][lb2[q]][1];
        // dots along the three modes, interleaved for ILP:
        //   sum_m sum_{j >= cend_m} That_m[i_m, j] xhat(u | m -> j)
        const int i0 = li0[q], i1 = li1[q];
        const int L0 = e0w - lce0[q], L1 = e1w - lce1[q], L2 = e2w - ce2;
        const double* d0 = dh + i0 + E * lce0[q];
        const double* d1 = dh + C::DHS + i1 + E * lce1[q];
        const double* d2 = dh + 2 * C::DHS + i2 + E * ce2;
        const double* x0 = xr + off + (lce0[q] - i0);
        const double* x1 = xr + off + E * (lce1[q] - i1);
        const double* x2 = xr + off + EE * (ce2 - i2);
        double ar0 = 0.0, ai0 = 0.0, ar1 = 0.0, ai1 = 0.0, ar2 = 0.0, ai2 = 0.0;
        if (!kp) {  // all-1x1 tile: real arithmetic
#pragma unroll
          for (int t = 0; t < E - 1; ++t) {
            if (t < L0) ar0 = fma(d0[E * t], x0[t], ar0);
            if (t < L1) ar1 = fma(d1[E * t], x1[E * t], ar1);
            if (t < L2) ar2 = fma(d2[E * t], x2[EE * t], ar2);
          }
        } else {
          const int XI = C::OFF_XI - C::OFF_XR;
#pragma unroll
          for (int t = 0; t < E - 1; ++t) {
            if (t < L0) {
              const double cr = d0[E * t], ci = d0[EE + E * t], yr = x0[t], yi = x0[XI + t];
              ar0 = fma(cr, yr, ar0);
              ar0 = fma(-ci, yi, ar0);
              ai0 = fma(cr, yi, ai0);
              ai0 = fma(ci, yr, ai0);
            }
            if (t < L1) {
              const double cr = d1[E * t], ci = d1[EE + E * t], yr = x1[E * t], yi = x1[XI + E * t];
              ar1 = fma(cr, yr, ar1);
              ar1 = fma(-ci, yi, ar1);
              ai1 = fma(cr, yi, ai1);
              ai1 = fma(ci, yr, ai1);
            }
            if (t < L2) {
              const double cr = d2[E * t], ci = d2[EE + E * t], yr = x2[EE * t], yi = x2[XI + EE * t];
              ar2 = fma(cr, yr, ar2);
              ar2 = fma(-ci, yi, ar2);
              ai2 = fma(cr, yi, ai2);
              ai2 = fma(ci, yr, ai2);
            }
          }
        }
        const double rr = xr[off] - (ar0 + ar1 + ar2);
        const double ri = xi[off] - (ai0 + ai1 + ai2);
        const double den = mur * mur + mui * mui;
        double vr = 0.0, vi = 0.0;
        if (!(den > a.tiny * a.tiny)) {
          singular = true;
        } else {
          const double inv = 1.0 / den;
          vr = (rr * mur + ri * mui) * inv;
          vi = (ri * mur - rr * mui) * inv;
        }
        xr[off] = vr;
        xi[off] = vi;
        if (orbit2) {
          xr[soff] = vr;
          xi[soff] = -vi;
        }
      }
      __syncthreads();
    }
    if (singular)
      atomicMin(a.status, static_cast<int>(tg.lt < 0x7f7f7f7e ? tg.lt : 0x7f7f7f7e));

    mark(4);
    // ---- back to the Schur basis -------------------------------------------------
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      if (!(kp & (1 << m))) continue;
      const double* pm = pd + m * E * kPStride;
      const int nw = tg.npair[m] * EE;
      for (int w = tid; w < nw; w += L3_THREADS) {
        const int i = tg.prow[m][w >> (2 * LT)], n = w & (EE - 1);
        const int na = n & MSK, nb = n >> LT;
        int l, st;
        if (m == 0) l = l3off<LT>(i, na, nb), st = 1;
        else if (m == 1) l = l3off<LT>(na, i, nb), st = E;
        else l = l3off<LT>(na, nb, i), st = EE;
        const double* p = pm + i * kPStride + 4;
        const int l2 = l + st;
        const double ar = xr[l], ai = xi[l], br = xr[l2], bi = xi[l2];
        xr[l] = p[0] * ar - p[1] * ai + p[2] * br - p[3] * bi;
        xi[l] = p[0] * ai + p[1] * ar + p[2] * bi + p[3] * br;
        xr[l2] = p[4] * ar - p[5] * ai + p[6] * br - p[7] * bi;
        xi[l2] = p[4] * ai + p[5] * ar + p[6] * bi + p[7] * br;
      }
      __syncthreads();
    }

    mark(5);
    }
  scatter:
    // ---- scatter X_t, release --------------------------------------------------
    for (int l = tid; l < L3_T; l += L3_THREADS) {
      const int i0 = l & MSK, i1 = (l >> LT) & MSK, i2 = l >> (2 * LT);
      if (i0 < e0 && i1 < e1 && i2 < e2)
        (DIST ? tg.xb : a.X)[tg.gbase + i0 + i1 * a.stride[1] + i2 * a.stride[2]] = xr[l];
    }
    __syncthreads();
    if (tid == 0) {
      if (DIST && a.sys && tg.own > 0) {  // read by the lower slabs' GPUs
        __threadfence_system();
        st_release_sys(a.fs[tg.own] + tg.lt, a.epoch);
      } else {
        __threadfence();
        st_release((DIST ? a.fs[tg.own] : a.flags) + tg.lt, a.epoch);
      }
      if (a.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[tg.lt] = t;
      }
    }
    mark(6);
    if (a.prof && tid == 0) atomicAdd(a.prof + 8, 1ull);
  }
  if (a.prof && tid == 0)
    for (int k = 0; k < 8; ++k) atomicAdd(a.prof + k, ph[k]);
}

template <int LT>
cudaError_t launch_l3(const SolveArgs& a0, cudaStream_t st, SolveLaunchInfo* info) {
  using C = L3C<LT>;
  SolveArgs a = a0;
  const int bytes = C::BYTES;
  const bool dist = LT == 3 && (a.nslab > 1 || a.sys);
  auto k = dist ? solve_lap3_kernel<LT, LT == 3> : solve_lap3_kernel<LT, false>;
  int nsm = 0, occ = 0;
  if (cudaError_t e = kernel_setup(k, bytes, C::THREADS, &nsm, &occ); e != cudaSuccess) return e;
  int64_t grid = static_cast<int64_t>(nsm) * occ;
  if (grid > a.ntiles) grid = a.ntiles;
  if (info) *info = SolveLaunchInfo{static_cast<int>(grid), C::THREADS, bytes, occ};
  cudaError_t le = launch_pdl(k, static_cast<unsigned>(grid), C::THREADS, bytes, st, a);
  return le != cudaSuccess ? le : cudaGetLastError();
}

}  // namespace

TileCaps solve_lap3_caps(int lt) {
  const int e = 1 << lt;
  return TileCaps{e, e * e * e, e * e};
}

cudaError_t launch_solve_lap3(int lt, const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info) {
  if (a.ntiles <= 0) return cudaSuccess;
  return lt == 3 ? launch_l3<3>(a, st, info) : launch_l3<4>(a, st, info);
}

}  // namespace tsg
