// Eigen-decoupled fibre solve (K5): the reduced solve once every mode but
// one (f) has been moved into its real block-eigenbasis by the transforms.
//
// Operator on the transformed tensor (solve.h, FibreArgs):
//     sum_{s in S} Y x_s Lambda_s + Y x_f T_f = R,
// Lambda_s block diagonal (1x1 lambda, 2x2 [[a, w], [-w, a]]), T_f the
// quasi-triangular Schur factor of mode f.  A unit = one cell of every S mode
// = 2^k real fibres along f (k = its 2x2 cells).  Complex structure: for the
// 2x2 cell of one S mode, z = y_0 + i y_1 turns [[a, w], [-w, a]] into the
// scalar a - i w.  With several 2x2 cells the first one is the re/im pair
// and every further cell t is diagonalised by the butterfly
// (z_0, z_1) -> (z_0 + i z_1, z_0 - i z_1) (eigenvalues a_t - i w_t,
// a_t + i w_t); the other half of the patterns are complex conjugates and
// never formed.  Each of the 2^(k-1) complex fibres then solves
//     (T_f + sigma I) z = r,  sigma = sum of its cells' eigenvalues,
// by back substitution over the 1x1/2x2 cells of T_f (2x2: Cramer), and the
// inverse butterfly restores the real fibres.  Everything runs in place in
// shared memory: one HBM read of R and one write of X per element.
//
// Reference: the same equation the recursion laplace_recursive / lap_rec
// (laplace.hpp:134-195) solves; the decoupling replaces the d-dimensional
// dependency DAG by independent fibres.
#include <climits>
#include <map>
#include <mutex>
#include <utility>

// DMMA as a side-effect-free asm: the compiler may hoist the L2 loads of T_f
// of later k steps above earlier products (fibre_wide_kernel's update loop)
#define TSG_DMMA_VOLATILE 0
#include "common.cuh"
#include "solve.h"
#include "util.h"

namespace tsg {
namespace {

constexpr int kThreads = 256;
constexpr int kTsmemMax = 64;  // T_f staged in shared memory up to this extent

struct Blk {
  int64_t base;
  int w, kb, r_lo, ncol, njob;
  int64_t bstride[kFibreMaxS];
  double bre[kFibreMaxS], bim[kFibreMaxS];
  double sreal;
};

TSG_DEVINL int64_t goff(const Blk& B, int col, int i, int64_t sf, int64_t sc = 1) {
  const int r = col % B.w, b = col / B.w;
  int64_t o = B.base + r * sc + static_cast<int64_t>(i) * sf;
#pragma unroll
  for (int t = 0; t < kFibreMaxS; ++t)
    if (t < B.kb && ((b >> t) & 1)) o += B.bstride[t];
  return o;
}

// In-place butterfly of every complex bit of the block, forward (inv = 0)
// or inverse (inv = 1).  Quad (re0, im0, re1, im1) per (row, unit, bit).
TSG_DEVINL void butterflies(const FibreArgs& a, const Blk& B, double* Y, bool inv) {
  const int nf = a.nf, ncol = B.ncol;
  for (int t = 0; t < B.kb; ++t) {
    const int step = B.w << t;
    for (int e = threadIdx.x; e < nf * ncol; e += blockDim.x) {
      const int i = e / ncol, col = e - i * ncol;
      const int rl = col % B.w, b = col / B.w;
      if ((b >> t) & 1) continue;
      const FibreCell c0 = a.cell0[a.cellrow0[B.r_lo + rl]];
      int imo;
      if (c0.size == 2) {
        if (B.r_lo + rl != c0.start) continue;  // re row of the mode-0 pair
        imo = 1;
      } else {
        if (t == 0 || (b & 1)) continue;  // bit 0 is the re/im pair itself
        imo = B.w;
      }
      double* y = Y + static_cast<size_t>(i) * ncol;
      const double re0 = y[col], im0 = y[col + imo];
      const double re1 = y[col + step], im1 = y[col + step + imo];
      if (!inv) {
        y[col] = re0 - im1;
        y[col + imo] = im0 + re1;
        y[col + step] = re0 + im1;
        y[col + step + imo] = im0 - re1;
      } else {
        y[col] = 0.5 * (re0 + re1);
        y[col + imo] = 0.5 * (im0 + im1);
        y[col + step] = 0.5 * (im0 - im1);
        y[col + step + imo] = -0.5 * (re0 - re1);
      }
    }
    __syncthreads();
  }
}

// 1/q for q > 0 (a sum of squares): MUFU reciprocal estimate and three
// Newton steps, branch-free (the IEEE division's slow-path check is a call)
TSG_DEVINL double rcp_pos(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  double e = fma(-q, r, 1.0);
  r = fma(r, e, r);
  e = fma(-q, r, 1.0);
  r = fma(r, e, r);
  e = fma(-q, r, 1.0);
  return fma(r, e, r);
}

// Back substitution of one complex (or real, im < 0) fibre along f.
TSG_DEVINL void solve_job(const FibreArgs& a, const double* T, double* Y, int ncol, int re, int im,
                          double sr, double si, int64_t off_hint) {
  const int nf = a.nf;
  const bool cx = im >= 0;
  for (int i = nf - 1; i >= 0;) {
    const double* fc = a.fcell + 4 * i;
    if (fc[0] == 2.0) {  // rows (i - 1, i): a 2x2 cell of T_f
      const int i0 = i - 1;
      double ar = Y[i0 * ncol + re], ai = cx ? Y[i0 * ncol + im] : 0.0;
      double br = Y[i * ncol + re], bi = cx ? Y[i * ncol + im] : 0.0;
      const double* t0 = T + static_cast<size_t>(i0) * nf;
      const double* t1 = T + static_cast<size_t>(i) * nf;
      for (int j = i + 1; j < nf; ++j) {
        const double zr = Y[j * ncol + re], zi = cx ? Y[j * ncol + im] : 0.0;
        ar = fma(-t0[j], zr, ar);
        ai = fma(-t0[j], zi, ai);
        br = fma(-t1[j], zr, br);
        bi = fma(-t1[j], zi, bi);
      }
      // M = [[t00 + s, t01], [t10, t11 + s]] (complex s)
      const double m00r = t0[i0] + sr, m11r = t1[i] + sr, m01 = t0[i], m10 = t1[i0];
      const double detr = m00r * m11r - si * si - m01 * m10;
      const double deti = si * (m00r + m11r);
      // eigenvalues (a +- i w) + s of the cell: singular check
      const double ea = fc[1] + sr, ew = fc[2];
      const double e1 = hypot(ea, si + ew), e2 = hypot(ea, si - ew);
      if (fmin(e1, e2) <= a.tiny)
        atomicMin(a.status, static_cast<int>(off_hint < INT_MAX - 1 ? off_hint : INT_MAX - 1));
      // za = (m11 ra - m01 rb) / det, zb = (m00 rb - m10 ra) / det
      const double nar = m11r * ar - si * ai - m01 * br;
      const double nai = m11r * ai + si * ar - m01 * bi;
      const double nbr = m00r * br - si * bi - m10 * ar;
      const double nbi = m00r * bi + si * br - m10 * ai;
      const double dd = detr * detr + deti * deti;
      const double ir = detr / dd, ii = -deti / dd;
      Y[i0 * ncol + re] = nar * ir - nai * ii;
      Y[i * ncol + re] = nbr * ir - nbi * ii;
      if (cx) {
        Y[i0 * ncol + im] = nar * ii + nai * ir;
        Y[i * ncol + im] = nbr * ii + nbi * ir;
      }
      i -= 2;
    } else {
      double rr = Y[i * ncol + re], ri = cx ? Y[i * ncol + im] : 0.0;
      const double* ti = T + static_cast<size_t>(i) * nf;
      for (int j = i + 1; j < nf; ++j) {
        rr = fma(-ti[j], Y[j * ncol + re], rr);
        if (cx) ri = fma(-ti[j], Y[j * ncol + im], ri);
      }
      const double dr = ti[i] + sr, di = si;
      const double dd = dr * dr + di * di;
      if (sqrt(dd) <= a.tiny)
        atomicMin(a.status, static_cast<int>(off_hint < INT_MAX - 1 ? off_hint : INT_MAX - 1));
      Y[i * ncol + re] = (rr * dr + ri * di) / dd;
      if (cx) Y[i * ncol + im] = (ri * dr - rr * di) / dd;
      i -= 1;
    }
  }
}

__global__ void __launch_bounds__(kThreads) fibre_solve_kernel(const FibreArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int nf = a.nf;
  const bool tsm = nf <= kTsmemMax;
  double* sT = sm;
  double* Y = sm + (tsm ? nf * nf : 0);
  int* jobs = reinterpret_cast<int*>(Y + static_cast<size_t>(a.maxcol) * nf);
  __shared__ Blk B;
  __shared__ int64_t s_blk;
  __shared__ int s_cnt;
  pdl_wait();
  if (tsm)
    for (int e = threadIdx.x; e < nf * nf; e += blockDim.x) sT[e] = a.Tt[e];
  const double* T = tsm ? sT : a.Tt;
  for (;;) {
    if (threadIdx.x == 0) {
      s_blk = atomicAdd(a.counter, 1);
      s_cnt = 0;
    }
    __syncthreads();
    const int64_t blk = s_blk;
    if (blk >= a.nblocks) break;
    if (threadIdx.x == 0) {
      int64_t rest = blk / a.nchunk;
      const int q = static_cast<int>(blk - rest * a.nchunk);
      B.r_lo = a.chunk_lo[q];
      B.w = a.chunk_lo[q + 1] - B.r_lo;
      int64_t base = B.r_lo;
      int kb = 0;
      double sreal = 0.0;
      for (int s = 0; s < a.ns; ++s) {
        const int64_t nx = rest / a.ncell[s];
        const int c = static_cast<int>(rest - nx * a.ncell[s]);
        rest = nx;
        const FibreCell fc = a.cells[s][c];
        base += static_cast<int64_t>(fc.start) * a.sstride[s];
        if (fc.size == 2) {
          B.bstride[kb] = a.sstride[s];
          B.bre[kb] = fc.re;
          B.bim[kb] = fc.im;
          ++kb;
        } else {
          sreal += fc.re;
        }
      }
      B.base = base;
      B.kb = kb;
      B.sreal = sreal;
      B.ncol = B.w << kb;
    }
    __syncthreads();
    const int ncol = B.ncol, w = B.w;
    // load: rows of w contiguous mode-0 elements
    {
      const int nb = 1 << B.kb;
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int row = warp; row < nf * nb; row += nw) {
        const int i = row / nb, b = row - i * nb;
        const double* src = a.X + goff(B, b * w, i, a.sf);
        double* dst = Y + static_cast<size_t>(i) * ncol + b * w;
        for (int r = lane; r < w; r += 32) dst[r] = src[r];
      }
    }
    // job list (complex fibres: re column of each pattern; real units: the column)
    for (int col = threadIdx.x; col < ncol; col += blockDim.x) {
      const int rl = col % w, b = col / w;
      const FibreCell c0 = a.cell0[a.cellrow0[B.r_lo + rl]];
      const bool job = c0.size == 2 ? (B.r_lo + rl == c0.start) : (B.kb == 0 || !(b & 1));
      if (job) jobs[atomicAdd(&s_cnt, 1)] = col;
    }
    __syncthreads();
    butterflies(a, B, Y, false);
    const int njob = s_cnt;
    for (int j = threadIdx.x; j < njob; j += blockDim.x) {
      const int col = jobs[j];
      const int rl = col % w, b = col / w;
      const FibreCell c0 = a.cell0[a.cellrow0[B.r_lo + rl]];
      double sr = B.sreal + c0.re, si = 0.0;
      int im = -1;
      if (c0.size == 2) {
        si = -c0.im;
        im = col + 1;
      } else if (B.kb > 0) {
        im = col + w;
      }
      for (int t = 0; t < B.kb; ++t) {
        sr += B.bre[t];
        si += ((b >> t) & 1) ? B.bim[t] : -B.bim[t];
      }
      solve_job(a, T, Y, ncol, col, im, sr, si, goff(B, col, 0, a.sf));
    }
    __syncthreads();
    butterflies(a, B, Y, true);
    {
      const int nb = 1 << B.kb;
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int row = warp; row < nf * nb; row += nw) {
        const int i = row / nb, b = row - i * nb;
        double* dst = a.X + goff(B, b * w, i, a.sf);
        const double* src = Y + static_cast<size_t>(i) * ncol + b * w;
        for (int r = lane; r < w; r += 32) dst[r] = src[r];
      }
    }
    __syncthreads();
  }
  pdl_trigger();
}

// ---- small free modes (n_f <= 32): units in registers -----------------------
// Per block: units = the mode-0 cells of the chunk; unit u has 2^k columns
// (k = 2x2 cells among its mode-0 cell and the block's S' cells), local
// index l: bit 0 = the re/im pair, bit t >= 1 = the t-th further 2x2 cell.
// Butterflies run per (unit, row) on the unit's 2^k values in registers; each
// job (one complex fibre) keeps its n_f values in registers for the back
// substitution against T_f in shared memory.
constexpr int kMaxUnits = 128;
constexpr int kSmallThreads = 128;  // 170 registers at n_f = 24: three CTAs per SM

struct UnitTab {
  int n;               // units in the block
  int rl0[kMaxUnits];  // first chunk row
  int k[kMaxUnits];    // complex bits (0..5)
  int job0[kMaxUnits + 1];
  double sr[kMaxUnits], si[kMaxUnits];  // mode-0 cell contribution to sigma (si: -omega for a pair)
};

TSG_DEVINL int ucol(int l, int rl0, int pair0, int w) {
  return pair0 ? rl0 + (l & 1) + w * (l >> 1) : rl0 + w * l;
}

template <int K, bool INV>
TSG_DEVINL void unit_bfly_k(double* y, int rl0, int pair0, int w) {
  constexpr int NL = 1 << K;
  double v[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) v[l] = y[ucol(l, rl0, pair0, w)];
#pragma unroll
  for (int t = 1; t < K; ++t) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      if ((l & 1) || ((l >> t) & 1)) continue;
      const int l1 = l | (1 << t);
      const double re0 = v[l], im0 = v[l | 1], re1 = v[l1], im1 = v[l1 | 1];
      if (!INV) {
        v[l] = re0 - im1;
        v[l | 1] = im0 + re1;
        v[l1] = re0 + im1;
        v[l1 | 1] = im0 - re1;
      } else {
        // unnormalised: the K - 1 halvings are one exact scaling at the end
        v[l] = re0 + re1;
        v[l | 1] = im0 + im1;
        v[l1] = im0 - im1;
        v[l1 | 1] = re1 - re0;
      }
    }
  }
  constexpr double scale = INV ? 1.0 / static_cast<double>(1 << (K - 1)) : 1.0;
#pragma unroll
  for (int l = 0; l < NL; ++l) y[ucol(l, rl0, pair0, w)] = INV ? v[l] * scale : v[l];
}

template <bool INV>
TSG_DEVINL void unit_butterfly(double* Y, int ncol, int i, int rl0, int k, int pair0, int w) {
  double* y = Y + static_cast<size_t>(i) * ncol;
  switch (k) {
    case 2: unit_bfly_k<2, INV>(y, rl0, pair0, w); break;
    case 3: unit_bfly_k<3, INV>(y, rl0, pair0, w); break;
    case 4: unit_bfly_k<4, INV>(y, rl0, pair0, w); break;
    case 5: unit_bfly_k<5, INV>(y, rl0, pair0, w); break;
    default: break;
  }
}

// Right-looking back substitution with the fibre in registers: once z_j
// (or the 2x2 pair z_{j-1}, z_j) is final, its column of T_f is applied to
// every row above.  All indices are compile-time (NF <= 24 stays in
// registers at 128 per thread).
template <int NF>
TSG_DEVINL void solve_job_reg(const FibreArgs& a, const double* T, const double* fc, double* Y,
                              int ncol, int re, int im, double sr, double si, int64_t off_hint) {
  const int nf = a.nf;
  const bool cx = im >= 0;
  double zr[NF], zi[NF];
#pragma unroll
  for (int i = 0; i < NF; ++i) {
    zr[i] = i < nf ? Y[i * ncol + re] : 0.0;
    zi[i] = (i < nf && cx) ? Y[i * ncol + im] : 0.0;
  }
  bool bad = false;
#pragma unroll
  for (int j = NF - 1; j >= 0; --j) {
    if (j >= nf) continue;
    const double code = fc[3 * j];
    if (code == 1.0) continue;  // first row of a pair: solved with its second row
    if (code == 2.0 && j >= 1) {
      const double m00r = T[(j - 1) * NF + j - 1] + sr, m11r = T[j * NF + j] + sr;
      const double m01 = T[(j - 1) * NF + j], m10 = T[j * NF + j - 1];
      const double detr = m00r * m11r - si * si - m01 * m10, deti = si * (m00r + m11r);
      const double ea = fc[3 * j + 1] + sr, ew = fc[3 * j + 2];
      bad = bad || fmin(ea * ea + (si + ew) * (si + ew), ea * ea + (si - ew) * (si - ew)) <= a.tiny * a.tiny;
      const double ar = zr[j - 1], ai = zi[j - 1], rr = zr[j], ri = zi[j];
      const double nar = m11r * ar - si * ai - m01 * rr, nai = m11r * ai + si * ar - m01 * ri;
      const double nbr = m00r * rr - si * ri - m10 * ar, nbi = m00r * ri + si * rr - m10 * ai;
      const double idd = rcp_pos(detr * detr + deti * deti), ir = detr * idd, ii = -deti * idd;
      zr[j - 1] = nar * ir - nai * ii;
      zi[j - 1] = nar * ii + nai * ir;
      zr[j] = nbr * ir - nbi * ii;
      zi[j] = nbr * ii + nbi * ir;
#pragma unroll
      for (int i = 0; i < NF; ++i) {
        if (i < j - 1) {
          const double t1 = T[i * NF + j], t0 = T[i * NF + j - 1];
          zr[i] = fma(-t1, zr[j], fma(-t0, zr[j - 1], zr[i]));
          zi[i] = fma(-t1, zi[j], fma(-t0, zi[j - 1], zi[i]));
        }
      }
    } else {
      const double dr = T[j * NF + j] + sr, dd = dr * dr + si * si;
      bad = bad || dd <= a.tiny * a.tiny;
      const double idd = rcp_pos(dd);
      const double rr = zr[j], ri = zi[j];
      zr[j] = (rr * dr + ri * si) * idd;
      zi[j] = (ri * dr - rr * si) * idd;
#pragma unroll
      for (int i = 0; i < NF; ++i) {
        if (i < j) {
          const double t = T[i * NF + j];
          zr[i] = fma(-t, zr[j], zr[i]);
          zi[i] = fma(-t, zi[j], zi[i]);
        }
      }
    }
  }
  if (bad) atomicMin(a.status, static_cast<int>(off_hint < INT_MAX - 1 ? off_hint : INT_MAX - 1));
#pragma unroll
  for (int i = 0; i < NF; ++i) {
    if (i < nf) {
      Y[i * ncol + re] = zr[i];
      if (cx) Y[i * ncol + im] = zi[i];
    }
  }
}

// Block pipeline of the small kernel: while block n is solved, block n+1's
// geometry is decoded from shared-memory cell tables and its data and unit
// table stream in with cp.async (two buffers).
struct SmallBuf {
  Blk B;
  int64_t blk;
  int nunit;
  int job0[kMaxUnits + 1];
  int64_t pb[1 << kFibreMaxS];  // element offset of every pattern's run at row 0 of f
};

TSG_DEVINL void decode_block(const FibreArgs& a, const FibreCell* scell, const int* soff, int64_t blk,
                             Blk& B, int& nunit) {
  // 32-bit index arithmetic (the host keeps nblocks < 2^31)
  unsigned rest = static_cast<unsigned>(blk) / static_cast<unsigned>(a.nchunk);
  const int q = static_cast<int>(static_cast<unsigned>(blk) - rest * static_cast<unsigned>(a.nchunk));
  B.r_lo = a.chunk_lo[q];
  B.w = a.chunk_lo[q + 1] - B.r_lo;
  B.njob = a.chunk_u0[q];  // first unit of the chunk (reused field)
  nunit = a.chunk_u0[q + 1] - a.chunk_u0[q];
  // sreal: the 1x1 cells' share of the shift: their sum (Laplace) or
  // product (gsylv: eigenvalues of a Kronecker product)
  int64_t base = static_cast<int64_t>(B.r_lo) * a.sc;
  int kb = 0;
  double sreal = a.gs ? 1.0 : 0.0;
  for (int s = 0; s < a.ns; ++s) {
    const unsigned nx = rest / static_cast<unsigned>(a.ncell[s]);
    const int c = static_cast<int>(rest - nx * static_cast<unsigned>(a.ncell[s]));
    rest = nx;
    const FibreCell fc = scell ? scell[soff[s] + c] : a.cells[s][c];
    base += static_cast<int64_t>(fc.start) * a.sstride[s];
    if (fc.size == 2) {
      B.bstride[kb] = a.sstride[s];
      B.bre[kb] = fc.re;
      B.bim[kb] = fc.im;
      ++kb;
    } else {
      sreal = a.gs ? sreal * fc.re : sreal + fc.re;
    }
  }
  B.base = base;
  B.kb = kb;
  B.sreal = sreal;
  B.ncol = B.w << kb;
}

TSG_DEVINL void block_patterns(const Blk& B, int64_t* pb) {
  for (int b = 0; b < (1 << B.kb); ++b) {
    int64_t o = B.base;
    for (int t = 0; t < B.kb; ++t)
      if ((b >> t) & 1) o += B.bstride[t];
    pb[b] = o;
  }
}

// Rows of a block <-> shared memory: the run of w contiguous mode-0
// elements of (row i of f, pattern b) is at X + pb[b] + i * sf and at
// Y + i * pitch + b * w.  Each warp instruction moves 32 / wp runs
// (wp = w rounded up to a power of two, at most 32), no divisions.
template <bool LOAD>
TSG_DEVINL void rows_io(const FibreArgs& a, double* Y, int pitch, const int64_t* pb, int w, int kb) {
  const int nf = a.nf, nb = 1 << kb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  int lw = 0;
  while ((1 << lw) < w && lw < 5) ++lw;
  const int sub = lane >> lw, r0 = lane & ((1 << lw) - 1), rpi = 32 >> lw;
  const int step = nw * rpi;  // runs per sweep of all warps
  const int nrun = nf * nb;
  if (w <= 32) {
    // One element per lane and run.  A lane's runs keep their pattern b (or
    // cycle through nb / step of them), so a lane walks the rows of f with
    // two pointer increments per element: no index decode, no pattern-offset
    // lookup in the loop; four rows in flight per lane.
    (void)nrun;
    if (r0 >= w) return;
    const int rsub = warp * rpi + sub;  // this lane's first run (< step; step and nb are powers of two)
    const int64_t sf = a.sf;
    auto walk = [&](double* y, const double* x, int i0, int di) {
      const int64_t dx = static_cast<int64_t>(di) * sf;
      const int dy = di * pitch;
      int i = i0;
      for (; i + 3 * di < nf; i += 4 * di) {
        if (LOAD) {
          cp_async8(y, x, 8);
          cp_async8(y + dy, x + dx, 8);
          cp_async8(y + 2 * dy, x + 2 * dx, 8);
          cp_async8(y + 3 * dy, x + 3 * dx, 8);
        } else {
          const double v0 = y[0], v1 = y[dy], v2 = y[2 * dy], v3 = y[3 * dy];
          double* xo = const_cast<double*>(x);
          xo[0] = v0;
          xo[dx] = v1;
          xo[2 * dx] = v2;
          xo[3 * dx] = v3;
        }
        y += 4 * dy;
        x += 4 * dx;
      }
      for (; i < nf; i += di) {
        if (LOAD) cp_async8(y, x, 8);
        else *const_cast<double*>(x) = *y;
        y += dy;
        x += dx;
      }
    };
    if (nb >= step) {
      for (int b = rsub; b < nb; b += step) walk(Y + b * w + r0, a.X + pb[b] + r0, 0, 1);
    } else {
      const int b = rsub & (nb - 1), i0 = rsub >> kb;
      walk(Y + static_cast<size_t>(i0) * pitch + b * w + r0, a.X + pb[b] + static_cast<int64_t>(i0) * sf + r0, i0,
           step >> kb);
    }
    return;
  }
  for (int run = warp * rpi + sub; run < nrun; run += step) {
    const int i = run >> kb, b = run & (nb - 1);
    double* y = Y + static_cast<size_t>(i) * pitch + b * w;
    const double* x = a.X + pb[b] + static_cast<int64_t>(i) * a.sf;
    for (int r = r0; r < w; r += 1 << lw) {
      if (LOAD) cp_async8(y + r, x + r, 8);
      else *const_cast<double*>(x + r) = y[r];
    }
  }
}

// cp.async of a block's rows (8-byte granules: rows start at any element)
// and of its chunk's unit table
TSG_DEVINL void issue_block(const FibreArgs& a, const Blk& B, const int64_t* pb, int nunit, double* Y, int pitch,
                            FibreUnit* su) {
  rows_io<true>(a, Y, pitch, pb, B.w, B.kb);
  const char* src = reinterpret_cast<const char*>(a.units + B.njob);
  char* dst = reinterpret_cast<char*>(su);
  for (int e = threadIdx.x; e < nunit * static_cast<int>(sizeof(FibreUnit) / 8); e += blockDim.x)
    cp_async8(dst + 8 * e, src + 8 * e, 8);
  cp_async_commit();
}

template <int NF>
__global__ void __launch_bounds__(kSmallThreads, 2) fibre_small_kernel(const FibreArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int nf = a.nf;
  // shared rows of a block: an odd pitch (ncol | 1) keeps the per-row
  // butterflies (lanes over rows) free of bank conflicts
  const int ybuf = (a.maxcol + 1) * nf;
  double* sT = sm;                      // NF x NF, row-major, zero padded
  double* sfc = sT + NF * NF;           // per row: code, a, omega
  double* Ys[2] = {sfc + 3 * NF, sfc + 3 * NF + ybuf};
  FibreUnit* sus[2] = {reinterpret_cast<FibreUnit*>(Ys[1] + ybuf),
                       reinterpret_cast<FibreUnit*>(Ys[1] + ybuf) + kMaxUnits};
  FibreCell* scell = a.cell_smem ? reinterpret_cast<FibreCell*>(sus[1] + kMaxUnits) : nullptr;
  __shared__ SmallBuf SB[2];
  __shared__ int soff[kFibreMaxS + 1];
  __shared__ int64_t s_next;
  pdl_wait();
  for (int e = threadIdx.x; e < NF * NF; e += blockDim.x) {
    const int i = e / NF, j = e - i * NF;
    sT[e] = (i < nf && j < nf) ? a.Tt[i * nf + j] : 0.0;
  }
  for (int i = threadIdx.x; i < NF; i += blockDim.x) {
    sfc[3 * i] = i < nf ? a.fcell[4 * i] : 0.0;
    sfc[3 * i + 1] = i < nf ? a.fcell[4 * i + 1] : 0.0;
    sfc[3 * i + 2] = i < nf ? a.fcell[4 * i + 2] : 0.0;
  }
  if (threadIdx.x == 0) {
    int o = 0;
    for (int s = 0; s < a.ns; ++s) {
      soff[s] = o;
      o += a.ncell[s];
    }
    soff[a.ns] = o;
  }
  __syncthreads();
  if (scell)
    for (int s = 0; s < a.ns; ++s)
      for (int c = threadIdx.x; c < a.ncell[s]; c += blockDim.x) scell[soff[s] + c] = a.cells[s][c];
  if (threadIdx.x == 0) {
    const int64_t b0 = atomicAdd(a.counter, 1);
    SB[0].blk = b0;
    if (b0 < a.nblocks) {
      decode_block(a, nullptr, soff, b0, SB[0].B, SB[0].nunit);
      block_patterns(SB[0].B, SB[0].pb);
    }
  }
  __syncthreads();
  if (SB[0].blk < a.nblocks) issue_block(a, SB[0].B, SB[0].pb, SB[0].nunit, Ys[0], SB[0].B.ncol | 1, sus[0]);
  int cur = 0;
#if SMALL_PROF
  long long ph[14] = {};
#endif
  for (;;) {
    SmallBuf& C = SB[cur];
    if (C.blk >= a.nblocks) break;
#if SMALL_PROF
    long long t0 = clock64();
#endif
    // prefetch the next block into the other buffer
    SmallBuf& Nx = SB[cur ^ 1];
    if (threadIdx.x == 0) {
      const int64_t nb = atomicAdd(a.counter, 1);
      Nx.blk = nb;
      if (nb < a.nblocks) {
        decode_block(a, scell, soff, nb, Nx.B, Nx.nunit);
        block_patterns(Nx.B, Nx.pb);
      }
    }
    __syncthreads();
#if SMALL_PROF
    long long t1 = clock64();
    ph[0] += t1 - t0;
#endif
    const bool more = Nx.blk < a.nblocks;
    if (more) {
      issue_block(a, Nx.B, Nx.pb, Nx.nunit, Ys[cur ^ 1], Nx.B.ncol | 1, sus[cur ^ 1]);
#if SMALL_PROF
      ph[8] += clock64() - t1;  // issue of the next block's loads alone
#endif
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#if SMALL_PROF
    long long t2 = clock64();
    ph[1] += t2 - t1;
#endif
    const Blk& B = C.B;
    const int ncol = B.ncol | 1, w = B.w, kb = B.kb, nunit = C.nunit;  // ncol: the shared pitch
    double* Y = Ys[cur];
    const FibreUnit* su = sus[cur];
    if (threadIdx.x == 0) {
      const int c2 = 1 << kb, c1 = kb ? 1 << (kb - 1) : 1;
      for (int u = 0; u <= nunit; ++u) {
        const int npb = u < nunit ? su[u].npair_before : su[nunit - 1].npair_before + su[nunit - 1].pair0;
        C.job0[u] = npb * c2 + (u - npb) * c1;
      }
    }
    __syncthreads();
#if SMALL_PROF
    ph[9] += clock64() - t2;  // job table (thread 0) + barrier
    const long long t2b = clock64();
#endif
    for (int u = threadIdx.x >> 5; u < nunit; u += blockDim.x >> 5) {  // a warp per unit, lanes over rows
      const int k = kb + su[u].pair0;
      if (k < 2) continue;
      for (int i = threadIdx.x & 31; i < nf; i += 32) unit_butterfly<false>(Y, ncol, i, su[u].rl0, k, su[u].pair0, w);
    }
#if SMALL_PROF
    ph[10] += clock64() - t2b;  // this warp's forward butterflies (before the barrier)
#endif
    __syncthreads();
#if SMALL_PROF
    long long t3 = clock64();
    ph[2] += t3 - t2;
#endif
    const int njob = C.job0[nunit];
    for (int j = threadIdx.x; j < njob; j += blockDim.x) {
      int lo = 0, hi = nunit - 1;  // last unit with job0 <= j
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (C.job0[mid] <= j) lo = mid;
        else hi = mid - 1;
      }
      const int u = lo;
      const int pair0 = su[u].pair0, k = kb + pair0, rl0 = su[u].rl0;
      const int l = (j - C.job0[u]) << 1;
      const int re = ucol(l, rl0, pair0, w);
      const int im = k ? ucol(l | 1, rl0, pair0, w) : -1;
      double sr = B.sreal + su[u].sr, si = su[u].si;
      for (int t = 0; t < kb; ++t) {
        const int bit = pair0 ? t + 1 : t;
        sr += B.bre[t];
        si += ((l >> bit) & 1) ? B.bim[t] : -B.bim[t];
      }
      solve_job_reg<NF>(a, sT, sfc, Y, ncol, re, im, sr, si, goff(B, re, 0, a.sf));
    }
#if SMALL_PROF
    ph[11] += clock64() - t3;  // this warp's jobs (before the barrier)
#endif
    __syncthreads();
#if SMALL_PROF
    long long t4 = clock64();
    ph[3] += t4 - t3;
#endif
    for (int u = threadIdx.x >> 5; u < nunit; u += blockDim.x >> 5) {  // a warp per unit, lanes over rows
      const int k = kb + su[u].pair0;
      if (k < 2) continue;
      for (int i = threadIdx.x & 31; i < nf; i += 32) unit_butterfly<true>(Y, ncol, i, su[u].rl0, k, su[u].pair0, w);
    }
#if SMALL_PROF
    ph[12] += clock64() - t4;  // this warp's inverse butterflies (before the barrier)
#endif
    __syncthreads();
#if SMALL_PROF
    const long long t5 = clock64();
#endif
    rows_io<false>(a, Y, ncol, C.pb, w, kb);
#if SMALL_PROF
    ph[13] += clock64() - t5;  // this warp's stores (before the barrier)
#endif
    __syncthreads();
#if SMALL_PROF
    ph[4] += clock64() - t4;
    ph[6] += 1;
#endif
    cur ^= 1;
  }
#if SMALL_PROF
  if (a.prof && (threadIdx.x & 31) == 0) {
    for (int k = 0; k < 7; ++k) atomicAdd(a.prof + k, static_cast<unsigned long long>(ph[k]));
    // finer split in the slots the team kernel uses for its role histogram
    for (int k = 8; k < 14; ++k) atomicAdd(a.prof + k, static_cast<unsigned long long>(ph[k]));
  }
#endif
  pdl_trigger();
}

// ---- large free modes: blocked back substitution on DMMA ---------------------
// Rows of f are processed in blocks of <= 8 (never splitting a 2x2 cell,
// FibreArgs::rb), bottom-up.  Block [i0, i1): the update
//     Y[i0:i1, :] -= T_f[i0:i1, i1:nf] Y[i1:nf, :]
// runs on DMMA m8n8k4 over all columns of the shared tile (re and im parts
// are just columns: T_f is real), four independent accumulator chains per
// warp; then every job back-substitutes its <= 8 rows with its own shift.
constexpr int kBigThreads = 256;

template <bool GS>
__global__ void __launch_bounds__(kBigThreads, 2) fibre_big_kernel(const FibreArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int nf = a.nf;
  const int pitch = a.pitch;
  double* Y = sm;
  double* jsr = Y + static_cast<size_t>(nf) * pitch;
  double* jsi = jsr + a.maxcol;
  int* jre = reinterpret_cast<int*>(jsi + a.maxcol);
  int* jim = jre + a.maxcol;
  FibreUnit* su = reinterpret_cast<FibreUnit*>((reinterpret_cast<uintptr_t>(jim + a.maxcol) + 15) & ~uintptr_t{15});
  FibreCell* scell = a.cell_smem ? reinterpret_cast<FibreCell*>(su + kMaxUnits) : nullptr;
  __shared__ SmallBuf SB;
  __shared__ int soff[kFibreMaxS + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  pdl_wait();
  if (threadIdx.x == 0) {
    int o = 0;
    for (int s = 0; s < a.ns; ++s) {
      soff[s] = o;
      o += a.ncell[s];
    }
    soff[a.ns] = o;
  }
  __syncthreads();
  if (scell)
    for (int s = 0; s < a.ns; ++s)
      for (int c = threadIdx.x; c < a.ncell[s]; c += blockDim.x) scell[soff[s] + c] = a.cells[s][c];
  for (;;) {
    if (threadIdx.x == 0) {
      SB.blk = atomicAdd(a.counter, 1);
      if (SB.blk < a.nblocks) {
        decode_block(a, scell, soff, SB.blk, SB.B, SB.nunit);
        block_patterns(SB.B, SB.pb);
      }
    }
    __syncthreads();
    if (SB.blk >= a.nblocks) break;
    const Blk& B = SB.B;
    const int nunit = SB.nunit;
    issue_block(a, B, SB.pb, nunit, Y, pitch, su);
    cp_async_wait<0>();
    __syncthreads();
    const int ncol = B.ncol, w = B.w, kb = B.kb;
    if (threadIdx.x == 0) {
      const int c2 = 1 << kb, c1 = kb ? 1 << (kb - 1) : 1;
      for (int u = 0; u <= nunit; ++u) {
        const int npb = u < nunit ? su[u].npair_before : su[nunit - 1].npair_before + su[nunit - 1].pair0;
        SB.job0[u] = npb * c2 + (u - npb) * c1;
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nunit * nf; e += blockDim.x) {
      const int u = e / nf, i = e - u * nf;
      const int k = kb + su[u].pair0;
      if (k >= 2) unit_butterfly<false>(Y, pitch, i, su[u].rl0, k, su[u].pair0, w);
    }
    const int njob = SB.job0[nunit];
    for (int j = threadIdx.x; j < njob; j += blockDim.x) {
      int lo = 0, hi = nunit - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (SB.job0[mid] <= j) lo = mid;
        else hi = mid - 1;
      }
      const int u = lo;
      const int pair0 = su[u].pair0, k = kb + pair0, rl0 = su[u].rl0;
      const int l = (j - SB.job0[u]) << 1;
      jre[j] = ucol(l, rl0, pair0, w);
      jim[j] = k ? ucol(l | 1, rl0, pair0, w) : -1;
      double sr = B.sreal + su[u].sr, si = su[u].si;
      for (int t = 0; t < kb; ++t) {
        const int bit = pair0 ? t + 1 : t;
        sr += B.bre[t];
        si += ((l >> bit) & 1) ? B.bim[t] : -B.bim[t];
      }
      jsr[j] = sr;
      jsi[j] = si;
    }
    __syncthreads();
    const int ntile = (ncol + 7) >> 3;
    for (int rb = a.nrb - 1; rb >= 0; --rb) {
      const int i0 = a.rb[rb], i1 = a.rb[rb + 1];
      if (i1 < nf) {
        const int ra = i0 + g;
        const bool arow = ra < i1;
        const double* trow = a.Tt + static_cast<size_t>(arow ? ra : i0) * nf;
        for (int nt = warp; nt < ntile; nt += nw) {
          const int n0 = nt << 3;
          const int bc = n0 + g < ncol ? n0 + g : 0;
          const bool bok = n0 + g < ncol;
          double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
          for (int k = i1; k < nf; k += 16) {
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
              const int kk = k + 4 * ch;
              if (kk < nf) {
                const int kr = kk + t4;
                const bool kin = kr < nf;
                const double av = (arow && kin) ? __ldg(trow + kr) : 0.0;
                const double bv = (bok && kin) ? Y[static_cast<size_t>(kr) * pitch + bc] : 0.0;
                dmma(c[ch][0], c[ch][1], av, bv);
              }
            }
          }
          const double s0 = (c[0][0] + c[1][0]) + (c[2][0] + c[3][0]);
          const double s1 = (c[0][1] + c[1][1]) + (c[2][1] + c[3][1]);
          const int col = n0 + 2 * t4;
          if (arow) {
            double* yr = Y + static_cast<size_t>(ra) * pitch;
            if (col < ncol) yr[col] -= s0;
            if (col + 1 < ncol) yr[col + 1] -= s1;
          }
        }
        __syncthreads();
      }
      // per job: back substitution inside [i0, i1)
      for (int j = threadIdx.x; j < njob; j += blockDim.x) {
        const int re = jre[j], im = jim[j];
        const double sr = jsr[j], si = jsi[j];
        const bool cx = im >= 0;
        bool bad = false;
        for (int i = i1 - 1; i >= i0;) {
          const double* fc = a.fcell + 4 * i;
          const double* ti = a.Tt + static_cast<size_t>(i) * nf;
          if (fc[0] == 2.0 && i - 1 >= i0) {
            const int i0r = i - 1;
            const double* t0 = a.Tt + static_cast<size_t>(i0r) * nf;
            double ar = Y[i0r * pitch + re], ai = cx ? Y[i0r * pitch + im] : 0.0;
            double br = Y[i * pitch + re], bi = cx ? Y[i * pitch + im] : 0.0;
            for (int jj = i + 1; jj < i1; ++jj) {
              const double zr = Y[jj * pitch + re], zi = cx ? Y[jj * pitch + im] : 0.0;
              ar = fma(-t0[jj], zr, ar);
              ai = fma(-t0[jj], zi, ai);
              br = fma(-ti[jj], zr, br);
              bi = fma(-ti[jj], zi, bi);
            }
            const double m00r = t0[i0r] + sr, m11r = ti[i] + sr, m01 = t0[i], m10 = ti[i0r];
            const double detr = m00r * m11r - si * si - m01 * m10, deti = si * (m00r + m11r);
            const double ea = fc[1] + sr, ew = fc[2];
            bad = bad || fmin(hypot(ea, si + ew), hypot(ea, si - ew)) <= a.tiny;
            const double nar = m11r * ar - si * ai - m01 * br, nai = m11r * ai + si * ar - m01 * bi;
            const double nbr = m00r * br - si * bi - m10 * ar, nbi = m00r * bi + si * br - m10 * ai;
            const double dd = detr * detr + deti * deti, ir = detr / dd, ii = -deti / dd;
            Y[i0r * pitch + re] = nar * ir - nai * ii;
            Y[i * pitch + re] = nbr * ir - nbi * ii;
            if (cx) {
              Y[i0r * pitch + im] = nar * ii + nai * ir;
              Y[i * pitch + im] = nbr * ii + nbi * ir;
            }
            i -= 2;
          } else {
            double rr = Y[i * pitch + re], ri = cx ? Y[i * pitch + im] : 0.0;
            for (int jj = i + 1; jj < i1; ++jj) {
              const double zr = Y[jj * pitch + re];
              rr = fma(-ti[jj], zr, rr);
              if (cx) ri = fma(-ti[jj], Y[jj * pitch + im], ri);
            }
            const double dr = ti[i] + sr, dd = dr * dr + si * si;
            bad = bad || sqrt(dd) <= a.tiny;
            Y[i * pitch + re] = (rr * dr + ri * si) / dd;
            if (cx) Y[i * pitch + im] = (ri * dr - rr * si) / dd;
            i -= 1;
          }
        }
        if (bad) {
          const int64_t off = goff(B, re, i0, a.sf);
          atomicMin(a.status, static_cast<int>(off < INT_MAX - 1 ? off : INT_MAX - 1));
        }
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < nunit * nf; e += blockDim.x) {
      const int u = e / nf, i = e - u * nf;
      const int k = kb + su[u].pair0;
      if (k >= 2) unit_butterfly<true>(Y, pitch, i, su[u].rl0, k, su[u].pair0, w);
    }
    __syncthreads();
    {
      const int nb = 1 << kb;
      for (int row = warp; row < nf * nb; row += nw) {
        const int i = row / nb, b = row - i * nb;
        double* dst = a.X + goff(B, b * w, i, a.sf);
        const double* src = Y + static_cast<size_t>(i) * pitch + b * w;
        for (int r = lane; r < w; r += 32) dst[r] = src[r];
      }
    }
    __syncthreads();
  }
  pdl_trigger();
}

// ---- large free modes: leader/helper teams on DMMA ---------------------------
// A block (chunk of mode-0 cells x one cell of every other S mode, <= 32
// real columns of n_f rows) is staged in shared memory; its complex jobs are
// packed into groups of 16 column slots (a job's re and im columns never
// straddle two groups).  A team of three warps solves one group by blocked
// back substitution over super-blocks s of two 8-row blocks of T_f
// (lo = [i0, mid), hi = [mid, i1); never splitting a 2x2 cell), bottom-up,
// as a two-stage pipeline:
//   helpers (one per 8-row block of s):  Y[s] -= T_f[s, i1:nf] Y[i1:nf]
//     (DMMA; the part from the rows of s+1 right after s+1 is solved, the
//     rest one step early, while the leader substitutes s+1),
//   leader: the in-block substitution of s (scalar FP64 in registers,
//     16 lanes, one real column per lane).
// On sm_100a the FP64 scalar pipe and DMMA share a sub-partition's math
// pipe: a DFMA dependency chain on a sub-partition that also runs a DMMA
// stream slows from ~9 to ~260-780 cycles per op (tools/probe/fp64_contend.cu).
// So the leaders issue no DMMA and sit on sub-partition 0 (hardware warp
// slot = 0 mod 4), the helpers on sub-partitions 1-3.
#ifndef WIDE_PROF
#define WIDE_PROF 0
#endif
#ifndef SMALL_PROF
#define SMALL_PROF 0
#endif
#if WIDE_PROF
#define WP_T(v) const long long v = clock64()
#define WP_ADD(k, t0) (ph[k] += clock64() - (t0))
#else
#define WP_T(v)
#define WP_ADD(k, t0)
#endif
#ifndef SUB8_PRO
#define SUB8_PRO false
#endif
constexpr int kTeamWarps = 5;  // leader (two 16-column groups, 32 lanes) + four helpers
constexpr int kWideTeams = 1;
// five warps per CTA (two CTAs per SM); roles are given by hardware
// sub-partition (warp slot mod 4, read from %warpid): the leader on the
// lowest sub-partition, the helpers on the others
constexpr int kWideThreads = kTeamWarps * kWideTeams * 32;
constexpr int kWideSlots = 2 * kWideCols;
constexpr int kWideUnits = 32;  // mode-0 cells per block (<= kWideCols rows)
TSG_DEVINL void team_sync(int team) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(team + 1), "r"(kTeamWarps * 32) : "memory");
}

struct WideTab {
  int col[kWideSlots];   // smem column of the slot (-1: padding)
  int im[kWideSlots];    // re slot of a complex job: its im column; else -1
  int role[kWideSlots];  // 0: re of a complex job, 1: its im, 2: real job, 3: padding
  double sr[kWideSlots], si[kWideSlots];
  int nslot;
  int jre[kWideCols], jim[kWideCols];
  double jsr[kWideCols], jsi[kWideCols];
};

// In-block back substitution of <= 8 rows (z in registers, T the 8x8
// diagonal block in shared memory, row-major), one lane per real column: a
// complex job's re and im columns sit on two partner lanes (sgn = +1 on the
// re lane, -1 on the im lane) that exchange only what the complex divisions
// couple; a real job is its own partner with si = 0.  code: 2 bits per row
// (0: 1x1 cell, 1/2: first/second row of a 2x2 cell); code, nr and T are
// warp-uniform, so every lane runs every shuffle.  Returns "numerically
// singular" (|det| <= tiny ||M||_F for a shifted 2x2 cell, |d| <= tiny for
// a 1x1 cell).
TSG_DEVINL bool sub8c(double (&z)[8], int nr, unsigned code, int partner, double sgn, double sr, double si,
                      double t2, const double* T) {
  constexpr int R = 8;
  bool bad = false;
#pragma unroll
  for (int j = R - 1; j >= 0; --j) {
    if (j >= nr) continue;
    const unsigned c = (code >> (2 * j)) & 3u;
    if (c == 1u) continue;  // first row of a pair: solved with its second row
    if (c == 2u && j >= 1) {
      const double m00r = T[(j - 1) * R + j - 1] + sr, m11r = T[j * R + j] + sr;
      const double m01 = T[(j - 1) * R + j], m10 = T[j * R + j - 1];
      const double detr = m00r * m11r - si * si - m01 * m10, deti = si * (m00r + m11r);
      const double dd = detr * detr + deti * deti, idd = rcp_pos(dd);
      const double fro2 = m00r * m00r + m11r * m11r + m01 * m01 + m10 * m10 + 2.0 * si * si;
      bad = bad || dd <= t2 * fro2;
      const double pa = __shfl_sync(0xffffffffu, z[j - 1], partner);
      const double pb = __shfl_sync(0xffffffffu, z[j], partner);
      const double na = m11r * z[j - 1] - sgn * si * pa - m01 * z[j];
      const double nb = m00r * z[j] - sgn * si * pb - m10 * z[j - 1];
      const double npa = __shfl_sync(0xffffffffu, na, partner);
      const double npb = __shfl_sync(0xffffffffu, nb, partner);
      z[j - 1] = (na * detr + sgn * npa * deti) * idd;
      z[j] = (nb * detr + sgn * npb * deti) * idd;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r < j - 1) z[r] = fma(-T[r * R + j], z[j], fma(-T[r * R + j - 1], z[j - 1], z[r]));
    } else {
      const double dr = T[j * R + j] + sr;
      const double dd = dr * dr + si * si, idd = rcp_pos(dd);
      bad = bad || dd <= t2;
      const double p = __shfl_sync(0xffffffffu, z[j], partner);
      z[j] = (z[j] * dr + sgn * p * si) * idd;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r < j) z[r] = fma(-T[r * R + j], z[j], z[r]);
    }
  }
  return bad;
}

template <bool PRO>
TSG_DEVINL bool sub8(double (&z)[8], int nr, unsigned code, int partner, double sgn, double sr, double si,
                     double t2, const double* T) {
  if (!PRO) return sub8c(z, nr, code, partner, sgn, sr, si, t2, T);
  constexpr int R = 8;
  // the pivots first: independent of the data, so the eight reciprocals
  // overlap instead of sitting on the substitution chain.  1x1 row j:
  // d = T_jj + s, 1/|d|^2; second row of a 2x2 cell: the shifted cell's
  // determinant and 1/|det|^2.
  double pr[R], pi[R], pv[R];
  bool bad = false;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const bool two = ((code >> (2 * j)) & 3u) == 2u && j >= 1;
    const double djj = T[j * R + j] + sr;
    double q = djj * djj + si * si;
    pr[j] = djj;
    pi[j] = si;
    if (j >= 1) {
      const double m00r = T[(j - 1) * R + j - 1] + sr, m01 = T[(j - 1) * R + j], m10 = T[j * R + j - 1];
      const double detr = m00r * djj - si * si - m01 * m10, deti = si * (m00r + djj);
      const double q2 = detr * detr + deti * deti;
      const double fro2 = m00r * m00r + djj * djj + m01 * m01 + m10 * m10 + 2.0 * si * si;
      pr[j] = two ? detr : djj;
      pi[j] = two ? deti : si;
      const bool sing = two ? q2 <= t2 * fro2 : q <= t2;
      q = two ? q2 : q;
      const unsigned c = (code >> (2 * j)) & 3u;
      bad = bad || (j < nr && c != 1u && sing);
    } else {
      bad = bad || (nr > 0 && (code & 3u) == 0u && q <= t2);
    }
    pv[j] = rcp_pos(q);
  }
#pragma unroll
  for (int j = R - 1; j >= 0; --j) {
    if (j >= nr) continue;
    const unsigned c = (code >> (2 * j)) & 3u;
    if (c == 1u) continue;  // first row of a pair: solved with its second row
    if (c == 2u && j >= 1) {
      const double m00r = T[(j - 1) * R + j - 1] + sr, m11r = T[j * R + j] + sr;
      const double m01 = T[(j - 1) * R + j], m10 = T[j * R + j - 1];
      const double pa = __shfl_sync(0xffffffffu, z[j - 1], partner);
      const double pb = __shfl_sync(0xffffffffu, z[j], partner);
      const double na = m11r * z[j - 1] - sgn * si * pa - m01 * z[j];
      const double nb = m00r * z[j] - sgn * si * pb - m10 * z[j - 1];
      const double npa = __shfl_sync(0xffffffffu, na, partner);
      const double npb = __shfl_sync(0xffffffffu, nb, partner);
      z[j - 1] = (na * pr[j] + sgn * npa * pi[j]) * pv[j];
      z[j] = (nb * pr[j] + sgn * npb * pi[j]) * pv[j];
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r < j - 1) z[r] = fma(-T[r * R + j], z[j], fma(-T[r * R + j - 1], z[j - 1], z[r]));
    } else {
      const double p = __shfl_sync(0xffffffffu, z[j], partner);
      z[j] = (z[j] * pr[j] + sgn * p * pi[j]) * pv[j];
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r < j) z[r] = fma(-T[r * R + j], z[j], z[r]);
    }
  }
  return bad;
}

// gsylv: in-block substitution of <= 8 rows of the pencil (S + z Tc) x = r
// (S quasi-triangular, Tc upper triangular, z = zr + i zi per job), same lane
// layout as sub8.  Right-looking: once x_j is final, r_k -= S_kj x_j +
// Tc_kj (z x_j) for k < j; w[j] returns this lane's component of z x_j (the
// coupling to the block above needs it).  The partner's component of x_j
// follows from the shuffled numerators, so z x_j costs no extra shuffle.
TSG_DEVINL bool sub8g(double (&x)[8], double (&wz)[8], int nr, unsigned code, int partner, double sgn, double zr,
                      double zi, double t2, const double* TS, const double* TC) {
  constexpr int R = 8;
  bool bad = false;
#pragma unroll
  for (int j = 0; j < R; ++j) wz[j] = 0.0;
#pragma unroll
  for (int j = R - 1; j >= 0; --j) {
    if (j >= nr) continue;
    const unsigned c = (code >> (2 * j)) & 3u;
    if (c == 1u) continue;  // first row of a pair: solved with its second row
    if (c == 2u && j >= 1) {
      const int j0 = j - 1;
      // M = S_cc + z Tc_cc (complex 2x2), entries (re, im)
      const double m00r = TS[j0 * R + j0] + zr * TC[j0 * R + j0], m00i = zi * TC[j0 * R + j0];
      const double m01r = TS[j0 * R + j] + zr * TC[j0 * R + j], m01i = zi * TC[j0 * R + j];
      const double m10r = TS[j * R + j0] + zr * TC[j * R + j0], m10i = zi * TC[j * R + j0];
      const double m11r = TS[j * R + j] + zr * TC[j * R + j], m11i = zi * TC[j * R + j];
      const double detr = (m00r * m11r - m00i * m11i) - (m01r * m10r - m01i * m10i);
      const double deti = (m00r * m11i + m00i * m11r) - (m01r * m10i + m01i * m10r);
      const double pa = __shfl_sync(0xffffffffu, x[j0], partner);
      const double pb = __shfl_sync(0xffffffffu, x[j], partner);
      // own component of (p + i q) y: p y_own - sgn q y_partner
      const double na = (m11r * x[j0] - sgn * m11i * pa) - (m01r * x[j] - sgn * m01i * pb);
      const double nb = (m00r * x[j] - sgn * m00i * pb) - (m10r * x[j0] - sgn * m10i * pa);
      const double npa = __shfl_sync(0xffffffffu, na, partner);
      const double npb = __shfl_sync(0xffffffffu, nb, partner);
      const double dd = detr * detr + deti * deti, idd = rcp_pos(dd);
      const double fro2 = m00r * m00r + m00i * m00i + m01r * m01r + m01i * m01i + m10r * m10r + m10i * m10i +
                          m11r * m11r + m11i * m11i;
      bad = bad || dd <= t2 * fro2;
      const double xa = (na * detr + sgn * npa * deti) * idd, xb = (nb * detr + sgn * npb * deti) * idd;
      const double xap = (npa * detr - sgn * na * deti) * idd, xbp = (npb * detr - sgn * nb * deti) * idd;
      x[j0] = xa;
      x[j] = xb;
      wz[j0] = zr * xa - sgn * zi * xap;
      wz[j] = zr * xb - sgn * zi * xbp;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r < j0)
          x[r] -= (TS[r * R + j0] * xa + TS[r * R + j] * xb) + (TC[r * R + j0] * wz[j0] + TC[r * R + j] * wz[j]);
    } else {
      const double mr = TS[j * R + j] + zr * TC[j * R + j], mi = zi * TC[j * R + j];
      const double p = __shfl_sync(0xffffffffu, x[j], partner);
      const double dd = mr * mr + mi * mi, idd = rcp_pos(dd);
      bad = bad || dd <= t2;
      const double xo = (x[j] * mr + sgn * p * mi) * idd, xp = (p * mr - sgn * x[j] * mi) * idd;
      x[j] = xo;
      wz[j] = zr * xo - sgn * zi * xp;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r < j) x[r] -= TS[r * R + j] * xo + TC[r * R + j] * wz[j];
    }
  }
  return bad;
}

// gsylv blocks: the free mode is mode 0 (contiguous fibres); column
// (pattern b, chunk row r) of the block is the fibre at X + pb[b] + r * sc.
template <bool LOAD>
TSG_DEVINL void gs_rows(const FibreArgs& a, double* Y, int pitch, const int64_t* pb, int w, int kb) {
  const int nf = a.nf, ncol = w << kb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int col = warp; col < ncol; col += nw) {
    const int b = col / w, r = col - b * w;
    const double* x = a.X + pb[b] + static_cast<int64_t>(r) * a.sc;
    for (int i = lane; i < nf; i += 32) {
      if (LOAD) cp_async8(Y + static_cast<size_t>(i) * pitch + col, x + i, 8);
      else *const_cast<double*>(x + i) = Y[static_cast<size_t>(i) * pitch + col];
    }
  }
}

// Rows of the block <-> shared memory: the run of w contiguous mode-0
// elements of (row i of f, pattern b) is at X + pb[b] + i * sf.  Each warp
// instruction moves 32 / wp such runs (wp = w rounded up to a power of two).
template <bool LOAD>
TSG_DEVINL void wide_rows(const FibreArgs& a, double* Y, int pitch, const int64_t* pb, int w, int kb) {
  const int nf = a.nf, nb = 1 << kb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  int lw = 0;
  while ((1 << lw) < w && lw < 5) ++lw;
  const int sub = lane >> lw, r = lane & ((1 << lw) - 1), rpi = 32 >> lw;
  if (r >= w) return;  // w <= kWideCols: one element per lane and run
  const int step = nw * rpi;  // rows of f per warp instruction sweep
  for (int b = 0; b < nb; ++b) {
    const int i_start = warp * rpi + sub;
    double* y = Y + static_cast<size_t>(i_start) * pitch + b * w + r;
    const double* x = a.X + pb[b] + static_cast<int64_t>(i_start) * a.sf + r;
    const int64_t xs = static_cast<int64_t>(step) * a.sf;
    for (int i = i_start; i < nf; i += step) {
      if (LOAD) cp_async8(y, x, 8);
      else *const_cast<double*>(x) = *y;
      y += step * pitch;
      x += xs;
    }
  }
}

// Shared-memory layout: Y (n_f x pitch), then per super-block s three 8x8
// blocks of T_f, row-major: [0] T[lo, lo], [1] T[hi, hi], [2] T[lo, hi]
// (zero padded), then the unit table and the optional S' cell table.
template <bool GS>
__global__ void __launch_bounds__(kWideThreads, 2) fibre_wide_kernel(const FibreArgs a) {
  constexpr int TDS = GS ? 384 : 192;  // Td doubles per super-block (gsylv: S blocks, then Tc blocks)
  extern __shared__ __align__(16) double sm[];
  const int nf = a.nf;
  const int pitch = a.pitch;
  const int zcol = pitch - 1;  // never written by a block: reads of padding slots give 0
  const int nsb = (a.nrb + 1) >> 1;
  double* Y = sm;
  double* Td = Y + static_cast<size_t>(nf) * pitch;
  FibreUnit* su = reinterpret_cast<FibreUnit*>(Td + TDS * static_cast<size_t>(nsb));
  FibreCell* scell = a.cell_smem ? reinterpret_cast<FibreCell*>(su + kWideUnits) : nullptr;
  __shared__ SmallBuf SB;
  __shared__ WideTab W;
  __shared__ int64_t pb[1 << kFibreMaxS];
  __shared__ int soff[kFibreMaxS + 1];
  __shared__ int hwslot[kWideThreads / 32], wrole[kWideThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  pdl_wait();
  if (threadIdx.x == 0) {
    int o = 0;
    for (int s = 0; s < a.ns; ++s) {
      soff[s] = o;
      o += a.ncell[s];
    }
    soff[a.ns] = o;
  }
  if (lane == 0) {
    unsigned hw;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(hw));
    hwslot[warp] = static_cast<int>(hw);
  }
  for (int i = threadIdx.x; i < nf; i += blockDim.x) Y[static_cast<size_t>(i) * pitch + zcol] = 0.0;
  for (int e = threadIdx.x; e < TDS * nsb; e += blockDim.x) {
    const int sb = e / TDS, ee = e % TDS, mat = ee / 192, part = (ee / 64) % 3, r = (e >> 3) & 7, c = e & 7;
    const int lo0 = a.rb[2 * sb], mid = a.rb[2 * sb + 1], hi1 = 2 * sb + 1 < a.nrb ? a.rb[2 * sb + 2] : mid;
    const int i = (part == 1 ? mid : lo0) + r, j = (part == 0 ? lo0 : mid) + c;
    const int ie = part == 1 ? hi1 : mid, je = part == 0 ? mid : hi1;
    const double* src = mat ? a.Tct : a.Tt;
    Td[e] = (i < ie && j < je) ? src[static_cast<size_t>(i) * nf + j] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // role = team rank (0 leader, 1..4 helpers) by sub-partition, or -1 (loads/stores only)
    int ord[kWideThreads / 32];
    for (int i = 0; i < nw; ++i) ord[i] = i;
    for (int i = 1; i < nw; ++i)  // by sub-partition, stable
      for (int j = i; j > 0 && (hwslot[ord[j]] & 3) < (hwslot[ord[j - 1]] & 3); --j) {
        const int t = ord[j];
        ord[j] = ord[j - 1];
        ord[j - 1] = t;
      }
    for (int i = 0; i < nw; ++i) wrole[i] = i < kTeamWarps ? 0 : -1;
    for (int i = 0; i < kTeamWarps && i < nw; ++i) wrole[ord[i]] = i;  // ord[0]: the leader
  }
  if (scell)
    for (int s = 0; s < a.ns; ++s)
      for (int c = threadIdx.x; c < a.ncell[s]; c += blockDim.x) scell[soff[s] + c] = a.cells[s][c];
  int64_t badoff = LLONG_MAX;
#if WIDE_PROF
  long long ph[12] = {};
#endif
  const double t2 = a.tiny * a.tiny;
  for (;;) {
    WP_T(tq);
    if (threadIdx.x == 0) {
      SB.blk = atomicAdd(a.counter, 1);
      if (SB.blk < a.nblocks) decode_block(a, scell, soff, SB.blk, SB.B, SB.nunit);
    }
    __syncthreads();
    if (SB.blk >= a.nblocks) break;
    const Blk& B = SB.B;
    const int nunit = SB.nunit;
    const int w = B.w, kb = B.kb, nb = 1 << kb;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      int64_t o = B.base;
      for (int t = 0; t < kb; ++t)
        if ((b >> t) & 1) o += B.bstride[t];
      pb[b] = o;
    }
    {
      const char* src = reinterpret_cast<const char*>(a.units + B.njob);
      char* dst = reinterpret_cast<char*>(su);
      for (int e = threadIdx.x; e < nunit * static_cast<int>(sizeof(FibreUnit) / 8); e += blockDim.x)
        cp_async8(dst + 8 * e, src + 8 * e, 8);
    }
    __syncthreads();
    if (GS) gs_rows<true>(a, Y, pitch, pb, w, kb);
    else wide_rows<true>(a, Y, pitch, pb, w, kb);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    WP_ADD(0, tq);
    WP_T(tb);
    if (threadIdx.x == 0) {
      const int c2 = 1 << kb, c1 = kb ? 1 << (kb - 1) : 1;
      for (int u = 0; u <= nunit; ++u) {
        const int npb = u < nunit ? su[u].npair_before : su[nunit - 1].npair_before + su[nunit - 1].pair0;
        SB.job0[u] = npb * c2 + (u - npb) * c1;
      }
    }
    // forward butterflies (units with >= 2 complex bits)
    for (int u = 0; u < nunit; ++u) {
      const int k = kb + su[u].pair0;
      if (k < 2) continue;
      for (int i = threadIdx.x; i < nf; i += blockDim.x) unit_butterfly<false>(Y, pitch, i, su[u].rl0, k, su[u].pair0, w);
    }
    __syncthreads();
    const int njob = SB.job0[nunit];
    for (int j = threadIdx.x; j < njob; j += blockDim.x) {
      int lo = 0, hi = nunit - 1;
      while (lo < hi) {
        const int md = (lo + hi + 1) >> 1;
        if (SB.job0[md] <= j) lo = md;
        else hi = md - 1;
      }
      const int u = lo;
      const int pair0 = su[u].pair0, k = kb + pair0, rl0 = su[u].rl0;
      const int l = (j - SB.job0[u]) << 1;
      W.jre[j] = ucol(l, rl0, pair0, w);
      W.jim[j] = k ? ucol(l | 1, rl0, pair0, w) : -1;
      double sr, si;
      if (GS) {  // product of the cells' eigenvalues
        sr = B.sreal * su[u].sr;
        si = B.sreal * su[u].si;
        for (int t = 0; t < kb; ++t) {
          const int bit = pair0 ? t + 1 : t;
          const double er = B.bre[t], ei = ((l >> bit) & 1) ? B.bim[t] : -B.bim[t];
          const double nr = sr * er - si * ei;
          si = sr * ei + si * er;
          sr = nr;
        }
      } else {  // sum
        sr = B.sreal + su[u].sr;
        si = su[u].si;
        for (int t = 0; t < kb; ++t) {
          const int bit = pair0 ? t + 1 : t;
          sr += B.bre[t];
          si += ((l >> bit) & 1) ? B.bim[t] : -B.bim[t];
        }
      }
      W.jsr[j] = sr;
      W.jsi[j] = si;
    }
    __syncthreads();
    // pack the jobs into groups of 16 slots (a complex job never straddles)
    if (threadIdx.x == 0) {
      int s = 0;
      for (int j = 0; j < njob; ++j) {
        const bool cx = W.jim[j] >= 0;
        if (cx && (s & 1)) {  // complex jobs on even slots (a lane's two fragment columns)
          W.col[s] = -1;
          W.im[s] = -1;
          W.role[s] = 3;
          W.sr[s] = W.si[s] = 0.0;
          ++s;
        }
        W.col[s] = W.jre[j];
        W.im[s] = W.jim[j];
        W.role[s] = cx ? 0 : 2;
        W.sr[s] = W.jsr[j];
        W.si[s] = W.jsi[j];
        ++s;
        if (cx) {
          W.col[s] = W.jim[j];
          W.im[s] = -1;
          W.role[s] = 1;
          W.sr[s] = W.jsr[j];
          W.si[s] = W.jsi[j];
          ++s;
        }
      }
      for (; s & 15; ++s) {
        W.col[s] = -1;
        W.im[s] = -1;
        W.role[s] = 3;
        W.sr[s] = W.si[s] = 0.0;
      }
      W.nslot = s;
    }
    __syncthreads();
    WP_ADD(1, tb);
    const int ngrp = W.nslot >> 4;
    const int team = 0;
    const int tw = wrole[warp] < 0 ? kTeamWarps : wrole[warp];  // 0 leader, 1..4 helpers
    // groups in pairs: the leader takes group gp on lanes 0..15 and gp + 1 on
    // lanes 16..31; helper h (tw = 1 + h) the 8-row block (h & 1) of every
    // super-block of group gp + (h >> 1)
    for (int gp = 0; tw < kTeamWarps && gp < ngrp; gp += 2) {
      const int h = tw - 1;
      const int grp = tw == 0 ? gp + (lane >> 4) : gp + (h >> 1);
      const bool live = grp < ngrp;
      const int s0 = (live ? grp : gp) << 4;
      int cb0 = W.col[s0 + g], cb1 = W.col[s0 + 8 + g];  // B-fragment columns
      cb0 = cb0 >= 0 ? cb0 : zcol;
      cb1 = cb1 >= 0 ? cb1 : zcol;
      const int cw00 = W.col[s0 + 2 * t4], cw01 = W.col[s0 + 2 * t4 + 1];
      const int cw10 = W.col[s0 + 8 + 2 * t4], cw11 = W.col[s0 + 9 + 2 * t4];
      // leader: this lane's column
      const int sl = s0 + (lane & 15);
      const int role = live ? W.role[sl] : 3;
      const int mycol = role == 3 ? -1 : W.col[sl];
      const int partner = role == 0 ? lane + 1 : role == 1 ? lane - 1 : lane;
      const int js = role == 1 ? sl - 1 : sl;  // the job's slot (shift)
      const double sgn = role == 1 ? -1.0 : 1.0;
      const double mysr = role == 3 ? 0.0 : W.sr[js], mysi = (role == 0 || role == 1) ? W.si[js] : 0.0;
      const int hm = h & 1;     // helper: 8-row block 2 s + hm of every super-block s
      double c[2][2][2] = {};   // [n-tile][k parity][2]: partial of the next super-block (S / T_f)
      double cz[2][2][2] = {};  // gsylv: the same with Tc (scaled by z per column when written)
      double la[4], lt[4];      // A fragments of T_f (S) / Tc [rows, rows of s+1] (k = i1 + 4 t4 + st)
      // gsylv: z of the lane's fragment columns (slots 2 t4, 2 t4 + 1 of each n-tile)
      const bool fcx0 = GS && W.role[s0 + 2 * t4] == 0, fcx1 = GS && W.role[s0 + 8 + 2 * t4] == 0;
      const double z0r = GS ? W.sr[s0 + 2 * t4] : 0.0, z0i = GS ? W.si[s0 + 2 * t4] : 0.0;
      const double z1r = GS ? W.sr[s0 + 2 * t4 + 1] : 0.0;
      const double z2r = GS ? W.sr[s0 + 8 + 2 * t4] : 0.0, z2i = GS ? W.si[s0 + 8 + 2 * t4] : 0.0;
      const double z3r = GS ? W.sr[s0 + 9 + 2 * t4] : 0.0;
      for (int q = nsb - 1; q >= 0; --q) {
        const int i0 = a.rb[2 * q], mid = a.rb[2 * q + 1];
        const int i1 = 2 * q + 1 < a.nrb ? a.rb[2 * q + 2] : mid;
        WP_T(tA);
        team_sync(team);  // rows >= i1 final
        WP_ADD(2, tA);
        if (tw > 0 && live) {
          // finish Y[block] -= T_f[block, i1:nf] Y[i1:nf]: the rows of s+1, then write
          const int r0 = hm == 0 ? i0 : mid, r1 = hm == 0 ? mid : i1;
          if (r0 < r1 && i1 < nf) {
            const int i2 = a.rb[min(2 * q + 4, a.nrb)];
#pragma unroll
            for (int st = 0; st < 4; ++st) {
              const int kr = i1 + 4 * t4 + st;
              const bool kin = kr < i2;
              const double* yk = Y + static_cast<size_t>(kin ? kr : i1) * pitch;
              const double b0 = yk[kin ? cb0 : zcol], b1 = yk[kin ? cb1 : zcol];
              dmma(c[0][st & 1][0], c[0][st & 1][1], la[st], b0);
              dmma(c[1][st & 1][0], c[1][st & 1][1], la[st], b1);
              if (GS) {
                dmma(cz[0][st & 1][0], cz[0][st & 1][1], lt[st], b0);
                dmma(cz[1][st & 1][0], cz[1][st & 1][1], lt[st], b1);
              }
            }
            const int ra = r0 + g;
            if (ra < r1) {
              double u00 = c[0][0][0] + c[0][1][0], u01 = c[0][0][1] + c[0][1][1];
              double u10 = c[1][0][0] + c[1][1][0], u11 = c[1][0][1] + c[1][1][1];
              if (GS) {  // + z (Tc x): complex (re, im) pair or two real columns
                const double v00 = cz[0][0][0] + cz[0][1][0], v01 = cz[0][0][1] + cz[0][1][1];
                const double v10 = cz[1][0][0] + cz[1][1][0], v11 = cz[1][0][1] + cz[1][1][1];
                if (fcx0) {
                  u00 += z0r * v00 - z0i * v01;
                  u01 += z0r * v01 + z0i * v00;
                } else {
                  u00 += z0r * v00;
                  u01 += z1r * v01;
                }
                if (fcx1) {
                  u10 += z2r * v10 - z2i * v11;
                  u11 += z2r * v11 + z2i * v10;
                } else {
                  u10 += z2r * v10;
                  u11 += z3r * v11;
                }
              }
              double* yr = Y + static_cast<size_t>(ra) * pitch;
              if (cw00 >= 0) yr[cw00] -= u00;
              if (cw01 >= 0) yr[cw01] -= u01;
              if (cw10 >= 0) yr[cw10] -= u10;
              if (cw11 >= 0) yr[cw11] -= u11;
            }
          }
        }
        team_sync(team);  // Y[s] fully updated
        WP_T(tL);
        if (tw == 0) {
          // in-block substitution of super-block s: hi, lo -= T[lo, hi] hi, lo
          double zl[8], zh[8];
          const bool own = mycol >= 0;
          const int nl = mid - i0, nh = i1 - mid;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            zl[r] = (own && r < nl) ? Y[(i0 + r) * pitch + mycol] : 0.0;
            zh[r] = (own && r < nh) ? Y[(mid + r) * pitch + mycol] : 0.0;
          }
          const double* T3 = Td + TDS * q;
          bool bad = false;
          if (GS) {
            double wh[8], wl[8];
            if (nh > 0) {
              bad = sub8g(zh, wh, nh, a.rbcode[2 * q + 1], partner, sgn, mysr, mysi, t2, T3 + 64, T3 + 256);
#pragma unroll
              for (int r = 0; r < 8; ++r) {
                double acc = zl[r];
#pragma unroll
                for (int k = 0; k < 8; ++k) acc = fma(-T3[128 + r * 8 + k], zh[k], fma(-T3[320 + r * 8 + k], wh[k], acc));
                zl[r] = acc;
              }
            }
            bad = sub8g(zl, wl, nl, a.rbcode[2 * q], partner, sgn, mysr, mysi, t2, T3, T3 + 192) || bad;
          } else {
            if (nh > 0) {
              bad = sub8<SUB8_PRO>(zh, nh, a.rbcode[2 * q + 1], partner, sgn, mysr, mysi, t2, T3 + 64);
#pragma unroll
              for (int r = 0; r < 8; ++r) {
                double acc = zl[r];
#pragma unroll
                for (int k = 0; k < 8; ++k) acc = fma(-T3[128 + r * 8 + k], zh[k], acc);
                zl[r] = acc;
              }
            }
            bad = sub8<SUB8_PRO>(zl, nl, a.rbcode[2 * q], partner, sgn, mysr, mysi, t2, T3) || bad;
          }
          if (own) {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              if (r < nl) Y[(i0 + r) * pitch + mycol] = zl[r];
              if (r < nh) Y[(mid + r) * pitch + mycol] = zh[r];
            }
            if (bad) badoff = min(badoff, goff(B, mycol, i0, a.sf, a.sc));
          }
          WP_ADD(3, tL);
        } else if (q >= 1 && live) {
          // partial of super-block s-1 over the final rows k >= i1, and the A
          // fragments of its update from the rows of s (used next step)
          const int p0 = a.rb[2 * q - 2], pm = a.rb[2 * q - 1];
          const int r0 = hm == 0 ? p0 : pm, r1 = hm == 0 ? pm : i0;
          const int ra = r0 + g;
          const size_t roff = static_cast<size_t>(ra < r1 ? ra : p0) * nf;
          const double* trow = a.Tt + roff;
          const double* tcrow = GS ? a.Tct + roff : trow;
#pragma unroll
          for (int st = 0; st < 4; ++st) {
            const int kr = i0 + 4 * t4 + st;
            la[st] = kr < i1 ? __ldg(trow + kr) : 0.0;
            if (GS) lt[st] = kr < i1 ? __ldg(tcrow + kr) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 2; ++v) c[u][v][0] = c[u][v][1] = cz[u][v][0] = cz[u][v][1] = 0.0;
          if (r0 < r1) {
            const double* tp = trow + i1 + t4;
            const double* tq = tcrow + i1 + t4;
            const double* yp = Y + static_cast<size_t>(i1 + t4) * pitch;
            const int nk4 = (nf - i1) >> 2;
            int j = 0;
#pragma unroll 4
            for (; j + 1 < nk4; j += 2) {
              const double a0 = __ldg(tp + 4 * j), a1 = __ldg(tp + 4 * j + 4);
              const double* y0 = yp + 4 * j * pitch;
              const double* y1 = y0 + 4 * pitch;
              const double b00 = y0[cb0], b01 = y0[cb1], b10 = y1[cb0], b11 = y1[cb1];
              dmma(c[0][0][0], c[0][0][1], a0, b00);
              dmma(c[1][0][0], c[1][0][1], a0, b01);
              dmma(c[0][1][0], c[0][1][1], a1, b10);
              dmma(c[1][1][0], c[1][1][1], a1, b11);
              if (GS) {
                const double e0 = __ldg(tq + 4 * j), e1 = __ldg(tq + 4 * j + 4);
                dmma(cz[0][0][0], cz[0][0][1], e0, b00);
                dmma(cz[1][0][0], cz[1][0][1], e0, b01);
                dmma(cz[0][1][0], cz[0][1][1], e1, b10);
                dmma(cz[1][1][0], cz[1][1][1], e1, b11);
              }
            }
            for (; 4 * j < nf - i1; ++j) {  // last k4 step (rows >= nf read as 0)
              const bool kin = i1 + 4 * j + t4 < nf;
              const double a0 = kin ? __ldg(tp + 4 * j) : 0.0;
              const double* y0 = yp + static_cast<size_t>(kin ? 4 * j : 0) * pitch;
              const double b00 = y0[kin ? cb0 : zcol], b01 = y0[kin ? cb1 : zcol];
              dmma(c[0][0][0], c[0][0][1], a0, b00);
              dmma(c[1][0][0], c[1][0][1], a0, b01);
              if (GS) {
                const double e0 = kin ? __ldg(tq + 4 * j) : 0.0;
                dmma(cz[0][0][0], cz[0][0][1], e0, b00);
                dmma(cz[1][0][0], cz[1][0][1], e0, b01);
              }
            }
          }
          WP_ADD(4, tL);
        }
      }
      team_sync(team);  // the last leader substitution is visible
    }
    __syncthreads();
    WP_T(ts);
    for (int u = 0; u < nunit; ++u) {
      const int k = kb + su[u].pair0;
      if (k < 2) continue;
      for (int i = threadIdx.x; i < nf; i += blockDim.x) unit_butterfly<true>(Y, pitch, i, su[u].rl0, k, su[u].pair0, w);
    }
    __syncthreads();
    if (GS) gs_rows<false>(a, Y, pitch, pb, w, kb);
    else wide_rows<false>(a, Y, pitch, pb, w, kb);
    __syncthreads();
    WP_ADD(5, ts);
#if WIDE_PROF
    ph[6] += 1;
#endif
  }
#if WIDE_PROF
  if (a.prof && lane == 0) {
    for (int k = 0; k < 7; ++k) atomicAdd(a.prof + k, static_cast<unsigned long long>(ph[k]));
    // sub-partition histogram of leaders (8..11) and helpers (12..15)
    if (wrole[warp] >= 0) atomicAdd(a.prof + (wrole[warp] == 0 ? 8 : 12) + (hwslot[warp] & 3), 1ull);
  }
#endif
  if (badoff != LLONG_MAX) atomicMin(a.status, static_cast<int>(badoff < INT_MAX - 1 ? badoff : INT_MAX - 1));
  pdl_trigger();
}

template <typename K>
cudaError_t launch_k(K k, const FibreArgs& a, size_t smem, int device, cudaStream_t st,
                     SolveLaunchInfo* info, int threads = kThreads) {
  // per (kernel, device): the shared-memory opt-in, the SM count and occupancy
  (void)device;
  int nsm = 0, occ = 0;
  if (cudaError_t e = kernel_setup(k, smem, threads, &nsm, &occ); e != cudaSuccess) return e;
  int grid = nsm * occ;
  if (a.nblocks < grid) grid = static_cast<int>(a.nblocks > 0 ? a.nblocks : 1);
  if (info) *info = SolveLaunchInfo{grid, threads, static_cast<int>(smem), occ};
  return launch_pdl(k, grid, threads, smem, st, a);
}

template <int NF>
cudaError_t launch_small(const FibreArgs& a, int device, cudaStream_t st, SolveLaunchInfo* info) {
  const size_t smem = (static_cast<size_t>(NF) * NF + 3 * NF + 2 * static_cast<size_t>(a.maxcol + 1) * a.nf) * sizeof(double) +
                      2 * kMaxUnits * sizeof(FibreUnit) + (a.cell_smem ? a.cell_smem : 0) * sizeof(FibreCell);
  return launch_k(fibre_small_kernel<NF>, a, smem, device, st, info, kSmallThreads);
}

}  // namespace

int fibre_pitch(int maxcol) { return ((maxcol + 11) / 16) * 16 + 4; }
size_t fibre_big_smem(int nf, int maxcol, int cell_smem) {
  return static_cast<size_t>(nf) * fibre_pitch(maxcol) * sizeof(double) +
         static_cast<size_t>(maxcol) * (2 * sizeof(double) + 2 * sizeof(int)) + 16 +
         kMaxUnits * sizeof(FibreUnit) + static_cast<size_t>(cell_smem) * sizeof(FibreCell);
}

size_t fibre_wide_smem(int nf, int maxcol, int cell_smem, int nrb, int gs) {
  if (nrb <= 0) nrb = (nf + 6) / 7;  // bound on the 8-row blocks (a 2x2 cell may shorten one to 7)
  const size_t nsb = (nrb + 1) / 2;
  return (static_cast<size_t>(nf) * fibre_pitch(maxcol) + (gs ? 384 : 192) * nsb) * sizeof(double) +
         kWideUnits * sizeof(FibreUnit) + static_cast<size_t>(cell_smem) * sizeof(FibreCell);
}

bool fibre_small_ok(int nf, int chunk_w) { return nf <= 24 && chunk_w <= kMaxUnits; }

cudaError_t launch_fibre_solve(const FibreArgs& a, int device, cudaStream_t st, SolveLaunchInfo* info) {
  int wmax = a.maxcol;  // chunk width bound (maxcol = wmax << nsc)
  (void)wmax;
  if (a.nf <= 24 && a.small) {
    if (a.nf <= 8) return launch_small<8>(a, device, st, info);
    if (a.nf <= 16) return launch_small<16>(a, device, st, info);
    return launch_small<24>(a, device, st, info);
  }
  if (a.wide) {
    const size_t smem = fibre_wide_smem(a.nf, a.maxcol, a.cell_smem, a.nrb, a.gs);
    if (a.gs) return launch_k(fibre_wide_kernel<true>, a, smem, device, st, info, kWideThreads);
    return launch_k(fibre_wide_kernel<false>, a, smem, device, st, info, kWideThreads);
  }
  if (a.big) {
    const size_t smem = fibre_big_smem(a.nf, a.maxcol, a.cell_smem);
    return launch_k(fibre_big_kernel<false>, a, smem, device, st, info, kBigThreads);
  }
  const size_t smem = (static_cast<size_t>(a.nf <= kTsmemMax ? a.nf * a.nf : 0) +
                       static_cast<size_t>(a.maxcol) * a.nf) * sizeof(double) +
                      static_cast<size_t>(a.maxcol) * sizeof(int);
  return launch_k(fibre_solve_kernel, a, smem, device, st, info);
}

}  // namespace tsg
