// K2 + K3: the reduced (quasi-)triangular Schur-basis solve as ONE persistent
// dataflow kernel on sm_100a.
//
// Reference path replaced: laplace_recursive / lap_rec / lap_base
// (laplace.hpp:134-195) and gsylv_recursive / gs_rec / gsylv_base
// (gsylv.hpp:62-159), i.e. "split the largest mode, solve the trailing block,
// apply B1 -= X2 x_mu A_mu(lo:k, k:hi), solve the leading block" down to an
// assembled base system solved by block_back_substitution
// (kernels.hpp:179-261).  The solution of the reduced system is unique
// (PAPER.md:98, :343), so the GPU is free to choose the schedule; parity is
// on X.
//
// Schedule.  The tensor is cut into tiles (per-mode boundaries snapped off
// 2x2 Schur blocks with the split_index rule, sylvester.hpp:43-49).  In the
// reduced Kronecker-sum system a tile depends only on tiles that are later
// in exactly one mode, so the recursion tree flattens into a DAG whose
// critical path is sum_m p_m - d + 1 tiles.  Tiles are handed out in a
// topological order (hyperplane sum_m t_m descending) through an atomic
// queue; a CTA that takes tile t
//   1. gathers B~_t into shared memory,
//   2. applies the left-looking off-diagonal updates
//        acc -= T_m[t_m, s] x_m X(t | m -> s)   for every later tile s
//      on DMMA tensor cores (mma.sync m8n8k4 f64), waiting on each source
//      tile's release flag (farthest first, so waits are rare),
//   3. solves the tile's own quasi-triangular system in shared memory by a
//      wavefront over Schur cells (one 1x1/2x2 block per mode, <= 2^d coupled
//      unknowns), each cell in closed form: per-mode 2x2 eigen-butterflies
//      across the lanes of a lane group, one division by the eigenvalue sum,
//      inverse butterflies, plus one step of refinement in real arithmetic,
//   4. writes X_t in place over B~_t and releases its flag.
// Deadlock freedom: a CTA only waits on tiles dequeued before its own, and
// those are held by CTAs that are already running.
//
// gsylv (family 1).  X x_0 S + X x_0 Tc x_1 A_1 ... x_{d-1} A_{d-1} = B~.
// The product term is factored as the chain W_{d-1} = X x_{d-1} A_{d-1},
// W_m = W_{m+1} x_m A_m, V = W_1 (reference chain updates, gsylv.hpp:111-123).
// Every factor is upper (quasi-)triangular, so a tile of W_m depends on W_{m+1}
// tiles later along mode m only: the same one-mode-later DAG as Laplace.  Each
// tile stores X_t and its W_m(t) for the tiles before it; the base cell is the
// pencil unit S_cc (x) I + Tc_cc (x) K_cc, solved by diagonalising the tail
// blocks and one <=2x2 complex solve per tail eigen-index.
#include <climits>
#include <cstdint>
#include <cstdio>

#include "common.cuh"
#include "solve.h"
#include "solve_common.cuh"
#include "util.h"

namespace tsg {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

template <int D, int FAM>
struct Cfg {
  static constexpr int THREADS = kThreads;
  static constexpr int EMAX = (D == 2) ? 1024 : (FAM == 0 ? 4096 : 2048);
  static constexpr int MB = (D == 2) ? 4 : (D == 3 ? 2 : 1);  // e_m <= 8*MB
  static constexpr int NBW = (D == 2) ? 1 : (D == 3 ? 4 : (D == 4 ? 8 : 16));
  static constexpr int NMAX = 64 * NBW;                         // cross-section cap
  static constexpr int KC = (D == 2) ? 16 : (D <= 4 ? 8 : 4);   // K rows per chunk
  static constexpr int NSTAGE = 3;                              // cp.async ring depth
  static constexpr int LDB = NMAX + 4;                          // == 4 (mod 16)
  static constexpr int MPAD = 8 * MB;
  static constexpr int LDA = MPAD + 4;
  static constexpr int NWB = FAM == 0 ? 0 : D - 1;              // W buffers in smem
  static constexpr int UMAX = D > 5 ? (1 << (D - 5)) : 1;       // unknowns per lane
  static constexpr int STAGE_B = KC * LDB;
  static constexpr int STAGE_A = KC * LDA;
  static constexpr int DBLK = MPAD * MPAD;                      // diag block per mode
  // shared memory carve-up (doubles, then ints)
  static constexpr int OFF_ACC = 0;
  static constexpr int OFF_W = OFF_ACC + EMAX;
  static constexpr int OFF_B = OFF_W + NWB * EMAX;
  static constexpr int OFF_A = OFF_B + NSTAGE * STAGE_B;
  static constexpr int OFF_D = OFF_A + NSTAGE * STAGE_A;
  static constexpr int NDBLK = FAM == 0 ? D : D + 1;            // + Tc block for gsylv
  static constexpr int OFF_EIG = OFF_D + NDBLK * DBLK;          // eigen data of tile rows
  static constexpr int OFF_CS = OFF_EIG + D * MPAD * kEigStride; // int64 csoff[NMAX]
  static constexpr int DOUBLES = OFF_CS + NMAX;
  static constexpr int BYTES = DOUBLES * 8 + EMAX * 4 /*slot table u32*/;
};

struct TileGeom {
  int64_t lt;
  int64_t gbase;
  int start[kMaxOrder], ext[kMaxOrder], tco[kMaxOrder], tstride[kMaxOrder];
  int E;
  int nc[kMaxOrder];
  int ncell, H;
  int pm[kMaxOrder], kp;  // pair modes (have a 2x2 cell), count
  int pidx[kMaxOrder];    // index j of mode m in pm, or -1
  unsigned char cs[kMaxOrder][kMaxCells], cz[kMaxOrder][kMaxCells];
};

// ---------------------------------------------------------------------------
// Lane-group butterflies for the closed-form cell solves.
// Bit j of an unknown's local index selects row 0/1 of the 2x2 Schur block of
// pair mode pm[j]; bits < LB live across lanes (shfl_xor), the rest across
// the UMAX registers of one lane.
// ---------------------------------------------------------------------------
template <int U>
TSG_DEVINL void partner_c(const Cplx (&z)[U], Cplx (&pz)[U], int j, int LB) {
  if (j < LB) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      pz[u].re = __shfl_xor_sync(0xffffffffu, z[u].re, 1 << j);
      pz[u].im = __shfl_xor_sync(0xffffffffu, z[u].im, 1 << j);
    }
  } else {
#pragma unroll
    for (int u = 0; u < U; ++u) pz[u] = z[u ^ (1 << (j - LB))];
  }
}
template <int U>
TSG_DEVINL void partner_r(const double (&z)[U], double (&pz)[U], int j, int LB) {
  if (j < LB) {
#pragma unroll
    for (int u = 0; u < U; ++u) pz[u] = __shfl_xor_sync(0xffffffffu, z[u], 1 << j);
  } else {
#pragma unroll
    for (int u = 0; u < U; ++u) pz[u] = z[u ^ (1 << (j - LB))];
  }
}

template <int D, int FAM>
__global__ void __launch_bounds__(kThreads, 1) solve_kernel(SolveArgs a) {
  using C = Cfg<D, FAM>;
  extern __shared__ __align__(16) double smem[];
  __shared__ TileGeom tg;
  __shared__ int s_tile;
  double* acc = smem + C::OFF_ACC;
  double* wbuf = smem + C::OFF_W;  // wbuf + (m-1)*EMAX for m = 1..D-1 (gsylv)
  double* dblk = smem + C::OFF_D;  // D diag blocks (+ Tc block for gsylv)
  double* seig = smem + C::OFF_EIG;
  // slot table of the (D-1)-mode cell grid: packed cell coordinates (5 bits
  // per mode) in the low bits, coordinate sum in bits 26..31.
  unsigned* slots = reinterpret_cast<unsigned*>(smem + C::DOUBLES);
  const int tid = threadIdx.x;

  for (;;) {
    if (tid == 0) s_tile = atomicAdd(a.counter, 1);
    __syncthreads();
    const int qi = s_tile;
    if (qi >= a.ntiles) break;

    // ---- tile geometry: host-built per-mode tables, loaded in parallel ------
    if (tid < D) {
      int64_t rem = a.order[qi];
      int tm = 0;
      for (int m = 0; m <= tid; ++m) {
        tm = static_cast<int>(rem % a.ntiles_mode[m]);
        rem /= a.ntiles_mode[m];
      }
      const TileMode& src = a.tmode[tid][tm];
      tg.tco[tid] = tm;
      tg.start[tid] = src.start;
      tg.ext[tid] = src.ext;
      tg.nc[tid] = src.nc;
      tg.pidx[tid] = src.pair;  // temporarily: pair flag
      for (int k = 0; k < src.nc; ++k) {
        tg.cs[tid][k] = src.cs[k];
        tg.cz[tid][k] = src.cz[k];
      }
    }
    __syncthreads();
    if (tid == 0) {
      int64_t lt = 0, mul = 1, gb = 0;
      int E = 1, H = 0, kp = 0, S = 1;
      for (int m = 0; m < D; ++m) {
        lt += tg.tco[m] * mul;
        mul *= a.ntiles_mode[m];
        tg.tstride[m] = E;
        E *= tg.ext[m];
        gb += static_cast<int64_t>(tg.start[m]) * a.stride[m];
        H += tg.nc[m] - 1;
        if (m < D - 1) S *= tg.nc[m];
        const bool pair = tg.pidx[m] != 0;
        tg.pidx[m] = pair ? kp : -1;
        if (pair) tg.pm[kp++] = m;
      }
      tg.lt = lt;
      tg.E = E;
      tg.gbase = gb;
      tg.H = H;
      tg.kp = kp;
      tg.ncell = S;  // slots of the (D-1)-mode grid
    }
    __syncthreads();
    const int E = tg.E;

    // ---- gather B~_t, stage diagonal blocks + eigen data, slot table ---------
    for (int l = tid; l < E; l += kThreads) {
      int rem = l;
      int64_t off = tg.gbase;
#pragma unroll
      for (int v = 0; v < D; ++v) {
        const int iv = rem % tg.ext[v];
        rem /= tg.ext[v];
        off += static_cast<int64_t>(iv) * a.stride[v];
      }
      cp_async8(acc + l, a.X + off, 8);
    }
    cp_async_commit();
    for (int m = 0; m < D; ++m) {
      const int em = tg.ext[m], st = tg.start[m], nm = a.dims[m];
      for (int e = tid; e < em * kEigStride; e += kThreads)
        seig[m * C::MPAD * kEigStride + e] = a.eig[m][static_cast<int64_t>(st) * kEigStride + e];
      for (int e = tid; e < em * em; e += kThreads) {
        const int i = e % em, j = e / em;
        dblk[m * C::DBLK + e] = a.T[m][(st + i) + static_cast<int64_t>(st + j) * nm];
      }
    }
    if (FAM == 1) {
      const int em = tg.ext[0], st = tg.start[0], nm = a.dims[0];
      for (int e = tid; e < em * em; e += kThreads) {
        const int i = e % em, j = e / em;
        dblk[D * C::DBLK + e] = a.Tc[(st + i) + static_cast<int64_t>(st + j) * nm];
      }
      for (int e = tid; e < C::NWB * E; e += kThreads) wbuf[(e / E) * C::EMAX + (e % E)] = 0.0;
    }
    for (int sl = tid; sl < tg.ncell; sl += kThreads) {
      int rem = sl;
      unsigned packed = 0, sum = 0;
#pragma unroll
      for (int v = 0; v < D - 1; ++v) {
        const int cv = rem % tg.nc[v];
        rem /= tg.nc[v];
        packed |= static_cast<unsigned>(cv) << (5 * v);
        sum += cv;
      }
      slots[sl] = packed | (sum << 26);
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- left-looking off-diagonal updates (DMMA) --------------------------
    // Far tiles (t_m+2 ..) of every mode first: they finished hyperplanes
    // ago; then the nearest neighbours, which are the last to be released.
    for (int part = 0; part < 2; ++part) {
      int64_t mul = 1;
      for (int m = 0; m < D; ++m) {
        const int tm = tg.tco[m], pm = a.ntiles_mode[m];
        const int* bm = a.bnd[m];
        int k_lo = 0, k_hi = 0, wt = -1;
        if (part == 0 && tm + 2 < pm) {
          k_lo = bm[tm + 2];
          k_hi = a.dims[m];
          wt = tm + 2;
        } else if (part == 1 && tm + 1 < pm) {
          k_lo = bm[tm + 1];
          k_hi = bm[tm + 2];
          wt = tm + 1;
        }
        if (wt >= 0) {
          const int64_t wtile = tg.lt + static_cast<int64_t>(wt - tm) * mul;
          if (FAM == 0) {
            update_pass<D, C>(a, tg, smem, acc, m, k_lo, k_hi, wtile, a.T[m], a.X, nullptr,
                                nullptr, 1, -1.0);
          } else if (m == 0) {
            // acc -= S[t0, later] x_0 X  +  Tc[t0, later] x_0 V
            update_pass<D, C>(a, tg, smem, acc, 0, k_lo, k_hi, wtile, a.T[0], a.X, a.Tc,
                                a.W[1], 2, -1.0);
          } else {
            // W'_m += A_m[t_m, later] x_m W_{m+1}   (W_D == X)
            update_pass<D, C>(a, tg, smem, wbuf + (m - 1) * C::EMAX, m, k_lo, k_hi, wtile,
                                a.T[m], m == D - 1 ? a.X : a.W[m + 1], nullptr, nullptr, 1, 1.0);
          }
        }
        mul *= pm;
      }
    }
    __syncthreads();

    // ---- in-tile wavefront over Schur cells --------------------------------
    // Hyperplane h = sum_m c_m from high to low.  Lane groups map onto the
    // slots of the (D-1)-mode cell grid; the last coordinate follows from h.
    {
      const int kp = tg.kp;
      const int LB = kp < 5 ? kp : 5;
      const int G = 1 << LB;
      const int NG = kThreads / G;
      const int gid = tid / G, lig = tid & (G - 1);
      const int U = 1 << (kp > 5 ? kp - 5 : 0);
      const int nlast = tg.nc[D - 1];
      const int rounds = (tg.ncell + NG - 1) / NG;
      for (int h = (a.dbg & 1) ? -1 : tg.H; h >= 0; --h) {
        for (int rd = 0; rd < rounds; ++rd) {
          const int slot = rd * NG + gid;
          int c[D];
          bool gvalid = slot < tg.ncell;
          {
            const unsigned pk = gvalid ? slots[slot] : 0u;
#pragma unroll
            for (int v = 0; v < D - 1; ++v) c[v] = (pk >> (5 * v)) & 31;
            const int cl = h - static_cast<int>(pk >> 26);
            gvalid = gvalid && cl >= 0 && cl < nlast;
            c[D - 1] = gvalid ? cl : 0;
          }
          if (!__any_sync(0xffffffffu, gvalid)) continue;  // warp-uniform skip
          // Unknowns of this lane.
          int off[C::UMAX];
          bool present[C::UMAX];
          int loc[C::UMAX][D];  // tile-local coordinates
          int bitv[C::UMAX][D];
#pragma unroll
          for (int u = 0; u < C::UMAX; ++u) {
            const int bits = lig | (u << LB);
            bool pres = gvalid && (u < U);
            int o = 0;
#pragma unroll
            for (int v = 0; v < D; ++v) {
              const int pj = tg.pidx[v];
              const int b = pj >= 0 ? (bits >> pj) & 1 : 0;
              const int cz = tg.cz[v][c[v]];
              if (b && cz == 1) pres = false;
              const int iv = tg.cs[v][c[v]] + (cz == 2 ? b : 0);
              loc[u][v] = iv;
              bitv[u][v] = b;
              o += iv * tg.tstride[v];
            }
            present[u] = pres;
            off[u] = o;
          }
          // In-tile left-looking dot products along mode v on buffer `src`
          // (independent accumulators per mode and parity for ILP).
          auto dot_mode = [&](int u, int v, const double* blk, const double* src) -> double {
            const int em = tg.ext[v];
            const int iv = loc[u][v];
            const int jend = tg.cs[v][c[v]] + tg.cz[v][c[v]];
            const int ts = tg.tstride[v];
            const double* drow = blk + iv;
            const double* sp = src + off[u] - iv * ts;
            double s0 = 0.0, s1 = 0.0;
            int j = jend;
            for (; j + 1 < em; j += 2) {
              s0 = fma(drow[j * em], sp[j * ts], s0);
              s1 = fma(drow[(j + 1) * em], sp[(j + 1) * ts], s1);
            }
            if (j < em) s0 = fma(drow[j * em], sp[j * ts], s0);
            return s0 + s1;
          };
          double r[C::UMAX];
          if (FAM == 0) {
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) {
              double s = 0.0;
              if (present[u]) {
                double sv[D];
#pragma unroll
                for (int v = 0; v < D; ++v)
                  sv[v] = (a.dbg & 2) ? 0.0 : dot_mode(u, v, dblk + v * C::DBLK, acc);
                s = acc[off[u]];
#pragma unroll
                for (int v = 0; v < D; ++v) s -= sv[v];
              }
              r[u] = s;
            }
          }
          // gsylv: tail partials P_m (external + in-tile later cells).
          double P[C::UMAX][D];
          if (FAM == 1) {
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) {
#pragma unroll
              for (int v = 1; v < D; ++v) {
                double s = 0.0;
                if (present[u]) {
                  const double* srcb = (v == D - 1) ? acc : wbuf + v * C::EMAX;
                  s = wbuf[(v - 1) * C::EMAX + off[u]] + dot_mode(u, v, dblk + v * C::DBLK, srcb);
                }
                P[u][v] = s;
              }
            }
          }
          // y <- A_v,cc x_v y with the cell's diagonal block of `blk`.
          // Shuffles are issued whenever v is a pair mode of the tile
          // (tile-uniform), so groups holding 1x1 cells stay converged.
          auto cell_mode_apply = [&](double (&y)[C::UMAX], int v, const double* blk) {
            const int em = tg.ext[v];
            const int i0 = tg.cs[v][c[v]];
            const int j = tg.pidx[v];
            if (j >= 0) {
              double py[C::UMAX];
              partner_r<C::UMAX>(y, py, j, LB);
              if (tg.cz[v][c[v]] == 2) {
                const double a00 = blk[i0 + i0 * em], a01 = blk[i0 + (i0 + 1) * em];
                const double a10 = blk[(i0 + 1) + i0 * em], a11 = blk[(i0 + 1) + (i0 + 1) * em];
#pragma unroll
                for (int u = 0; u < C::UMAX; ++u)
                  y[u] = bitv[u][v] == 0 ? a00 * y[u] + a01 * py[u] : a10 * py[u] + a11 * y[u];
                return;
              }
            }
            const double d0 = blk[i0 + i0 * em];
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) y[u] *= d0;
          };
          // ---- closed-form cell solve in the real normal form -------------------
          // Every 2x2 diagonal block is W (alpha I + beta J) W^{-1} with real W
          // (J = [[0,1],[-1,0]]), or W diag(l0, l1) W^{-1} for a real pair.  In
          // the W basis, J is diagonalised by the FIXED butterfly
          //   zeta+ = (x0 - i x1)/2 (eigenvalue +i),  zeta- = (x0 + i x1)/2 (-i),
          // so the cell operator sum_v A_v,cc becomes diagonal with entries
          // s + i*omega (s, omega real sums over the modes).
          // wd layout (kEigStride doubles at a block's first row):
          //   [0] alpha|l0  [1] l1  [2] beta  [3] kind (0 1x1, 1 complex, 2 real)
          //   [4..7] W^{-1} (row-major)  [8..11] W (row-major)
          auto wd_of = [&](int v) -> const double* {
            return seig + (v * C::MPAD + tg.cs[v][c[v]]) * kEigStride;
          };
          // real 2x2 transform of mode v's pair (M row-major at wd + off4)
          auto pair_real = [&](double (&x)[C::UMAX], int v, int off4) {
            const int j = tg.pidx[v];
            if (j < 0) return;
            double px[C::UMAX];
            partner_r<C::UMAX>(x, px, j, LB);
            if (tg.cz[v][c[v]] != 2) return;
            const double* M = wd_of(v) + off4;
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u)
              x[u] = bitv[u][v] == 0 ? M[0] * x[u] + M[1] * px[u] : M[2] * px[u] + M[3] * x[u];
          };
          auto pair_fwd = [&](Cplx (&z)[C::UMAX], int v) {
            const int j = tg.pidx[v];
            if (j < 0) return;
            Cplx pz[C::UMAX];
            partner_c<C::UMAX>(z, pz, j, LB);
            if (tg.cz[v][c[v]] != 2 || wd_of(v)[3] != 1.0) return;
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) {
              // b=0: (z0 - i z1)/2 ; b=1: (z0 + i z1)/2 with z0 = partner
              const Cplx o = z[u], p = pz[u];
              z[u] = bitv[u][v] == 0 ? Cplx{0.5 * (o.re + p.im), 0.5 * (o.im - p.re)}
                                     : Cplx{0.5 * (p.re - o.im), 0.5 * (p.im + o.re)};
            }
          };
          auto pair_inv = [&](Cplx (&z)[C::UMAX], int v) {
            const int j = tg.pidx[v];
            if (j < 0) return;
            Cplx pz[C::UMAX];
            partner_c<C::UMAX>(z, pz, j, LB);
            if (tg.cz[v][c[v]] != 2 || wd_of(v)[3] != 1.0) return;
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) {
              // x0 = zeta+ + zeta- ; x1 = i (zeta+ - zeta-)
              const Cplx o = z[u], p = pz[u];
              z[u] = bitv[u][v] == 0 ? Cplx{o.re + p.re, o.im + p.im}
                                     : Cplx{o.im - p.im, p.re - o.re};
            }
          };
          // eigenvalue of mode v's cell block for unknown u (in the W basis)
          auto lam_of = [&](int u, int v) -> Cplx {
            const int i0 = tg.cs[v][c[v]];
            if (tg.cz[v][c[v]] == 2) {
              const double* w = wd_of(v);
              const int b = bitv[u][v];
              if (w[3] == 1.0) return Cplx{w[0], b ? -w[2] : w[2]};
              return Cplx{b ? w[1] : w[0], 0.0};
            }
            return Cplx{dblk[v * C::DBLK + i0 + i0 * tg.ext[v]], 0.0};
          };

          bool singular = false;
          // y = cellop^{-1} rhs (real in, real out).
          auto cell_solve = [&](const double (&rhs)[C::UMAX], double (&y)[C::UMAX]) {
            if (FAM == 0 && kp == 0) {  // all-1x1 tile: one real division
#pragma unroll
              for (int u = 0; u < C::UMAX; ++u) {
                double mu = 0.0;
#pragma unroll
                for (int v = 0; v < D; ++v) {
                  const int i0 = tg.cs[v][c[v]];
                  mu += dblk[v * C::DBLK + i0 + i0 * tg.ext[v]];
                }
                if (fabs(mu) <= a.tiny) {
                  singular = singular || present[u];
                  mu = 1.0;
                }
                y[u] = present[u] ? rhs[u] / mu : 0.0;
              }
              return;
            }
            const int v_first = (FAM == 0) ? 0 : 1;
            double x[C::UMAX];
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) x[u] = rhs[u];
#pragma unroll
            for (int v = v_first; v < D; ++v) pair_real(x, v, 4);  // W^{-1}
            Cplx z[C::UMAX];
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) z[u] = Cplx{x[u], 0.0};
#pragma unroll
            for (int v = v_first; v < D; ++v) pair_fwd(z, v);
            if (FAM == 0) {
#pragma unroll
              for (int u = 0; u < C::UMAX; ++u) {
                double sr = 0.0, si = 0.0;
#pragma unroll
                for (int v = 0; v < D; ++v) {
                  const Cplx l = lam_of(u, v);
                  sr += l.re;
                  si += l.im;
                }
                const double den = sr * sr + si * si;
                if (den <= a.tiny * a.tiny) {
                  singular = singular || present[u];
                  z[u] = Cplx{0.0, 0.0};
                } else {
                  const double inv = 1.0 / den;
                  z[u] = Cplx{(z[u].re * sr + z[u].im * si) * inv, (z[u].im * sr - z[u].re * si) * inv};
                }
              }
            } else {
              // mode-0 pencil unit (S_cc + kappa Tc_cc) per tail eigen-index
              const int e0 = tg.ext[0], i0 = tg.cs[0][c[0]];
              const double* Sb = dblk;
              const double* Tb = dblk + D * C::DBLK;
              const int j0 = tg.pidx[0];
              Cplx pz[C::UMAX];
              if (j0 >= 0) partner_c<C::UMAX>(z, pz, j0, LB);
              const bool two = tg.cz[0][c[0]] == 2;
#pragma unroll
              for (int u = 0; u < C::UMAX; ++u) {
                Cplx kappa{1.0, 0.0};
#pragma unroll
                for (int v = 1; v < D; ++v) kappa = cmul(kappa, lam_of(u, v));
                auto ent = [&](int r_, int c_) {
                  return cadd(Cplx{Sb[(i0 + r_) + (i0 + c_) * e0], 0.0},
                              cmul(kappa, Cplx{Tb[(i0 + r_) + (i0 + c_) * e0], 0.0}));
                };
                if (!two) {
                  Cplx dd = ent(0, 0);
                  if (fabs(dd.re) + fabs(dd.im) <= a.tiny) {
                    singular = singular || present[u];
                    dd = Cplx{1.0, 0.0};
                  }
                  z[u] = cdiv(z[u], dd);
                } else {
                  const Cplx m00 = ent(0, 0), m01 = ent(0, 1), m10 = ent(1, 0), m11 = ent(1, 1);
                  Cplx det = cadd(cmul(m00, m11), cmul(Cplx{-m01.re, -m01.im}, m10));
                  if (fabs(det.re) + fabs(det.im) <= a.tiny * a.tiny) {
                    singular = singular || present[u];
                    det = Cplx{1.0, 0.0};
                  }
                  const int b = bitv[u][0];
                  // x0 = (m11 r0 - m01 r1)/det ; x1 = (m00 r1 - m10 r0)/det
                  const Cplx r0 = b == 0 ? z[u] : pz[u];
                  const Cplx r1 = b == 0 ? pz[u] : z[u];
                  const Cplx num = b == 0 ? cadd(cmul(m11, r0), cmul(Cplx{-m01.re, -m01.im}, r1))
                                          : cadd(cmul(m00, r1), cmul(Cplx{-m10.re, -m10.im}, r0));
                  z[u] = cdiv(num, det);
                }
              }
            }
#pragma unroll
            for (int v = D - 1; v >= v_first; --v) pair_inv(z, v);
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) x[u] = z[u].re;
#pragma unroll
            for (int v = v_first; v < D; ++v) pair_real(x, v, 8);  // W
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) y[u] = present[u] ? x[u] : 0.0;
          };
          // Cell operator applied to y (real): Laplace sum_v y x_v D_v,cc;
          // gsylv y x_0 S_cc + (y x_tails A_cc) x_0 Tc_cc.
          auto cell_op = [&](const double (&y)[C::UMAX], double (&out)[C::UMAX]) {
            if (FAM == 0) {
#pragma unroll
              for (int u = 0; u < C::UMAX; ++u) out[u] = 0.0;
              for (int v = 0; v < D; ++v) {
                double t[C::UMAX];
#pragma unroll
                for (int u = 0; u < C::UMAX; ++u) t[u] = y[u];
                cell_mode_apply(t, v, dblk + v * C::DBLK);
#pragma unroll
                for (int u = 0; u < C::UMAX; ++u) out[u] += t[u];
              }
            } else {
              double t[C::UMAX], s[C::UMAX];
#pragma unroll
              for (int u = 0; u < C::UMAX; ++u) t[u] = s[u] = y[u];
              for (int v = D - 1; v >= 1; --v) cell_mode_apply(t, v, dblk + v * C::DBLK);
              cell_mode_apply(t, 0, dblk + D * C::DBLK);
              cell_mode_apply(s, 0, dblk);
#pragma unroll
              for (int u = 0; u < C::UMAX; ++u) out[u] = s[u] + t[u];
            }
          };

          if (FAM == 1) {
            // R = P_1 + A_1cc x_1 (P_2 + ... (P_{D-1}))  ;  rhs = acc - mode-0 dots - Tc_cc x_0 R
            double R[C::UMAX];
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) R[u] = P[u][D - 1];
            for (int v = D - 2; v >= 1; --v) {
              cell_mode_apply(R, v, dblk + v * C::DBLK);
#pragma unroll
              for (int u = 0; u < C::UMAX; ++u) R[u] += P[u][v];
            }
            cell_mode_apply(R, 0, dblk + D * C::DBLK);
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) {
              double s = 0.0;
              if (present[u]) {
                s = acc[off[u]] - R[u] - dot_mode(u, 0, dblk, acc) -
                    dot_mode(u, 0, dblk + D * C::DBLK, wbuf);  // W_1 == V
              }
              r[u] = s;
            }
          }

          double y[C::UMAX];
          cell_solve(r, y);
          if (a.refine) {  // plan-uniform: some 2x2 eigenbasis is ill-conditioned
            double res[C::UMAX], dy[C::UMAX];
            cell_op(y, res);
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) res[u] = present[u] ? r[u] - res[u] : 0.0;
            cell_solve(res, dy);
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) y[u] += dy[u];
          }

          if (singular && gvalid)
            atomicMin(a.status, static_cast<int>(tg.lt < 0x7f7f7f7e ? tg.lt : 0x7f7f7f7e));
#pragma unroll
          for (int u = 0; u < C::UMAX; ++u)
            if (present[u]) acc[off[u]] = y[u];
          if (FAM == 1) {
            // W_{D-1} = A_{D-1,cc} x_{D-1} y + P_{D-1}; W_m = A_m,cc x_m W_{m+1} + P_m
            double w[C::UMAX];
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) w[u] = y[u];
            for (int v = D - 1; v >= 1; --v) {
              cell_mode_apply(w, v, dblk + v * C::DBLK);
#pragma unroll
              for (int u = 0; u < C::UMAX; ++u) {
                w[u] += P[u][v];
                if (present[u]) wbuf[(v - 1) * C::EMAX + off[u]] = w[u];
              }
            }
          }
        }
        __syncthreads();
      }
    }

    // ---- scatter X_t (and W_m(t)), release -----------------------------------
    for (int l = tid; l < E; l += kThreads) {
      int rem = l;
      int64_t off = tg.gbase;
#pragma unroll
      for (int v = 0; v < D; ++v) {
        const int iv = rem % tg.ext[v];
        rem /= tg.ext[v];
        off += static_cast<int64_t>(iv) * a.stride[v];
      }
      a.X[off] = acc[l];
      if (FAM == 1) {
#pragma unroll
        for (int v = 1; v < D; ++v) a.W[v][off] = wbuf[(v - 1) * C::EMAX + l];
      }
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(a.flags + tg.lt, a.epoch);
    }
  }
}

template <int D, int FAM>
cudaError_t launch_t(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info) {
  using C = Cfg<D, FAM>;
  auto k = solve_kernel<D, FAM>;
  // smem opt-in and the persistent grid size (per device)
  int nsm = 0, occ = 0;
  if (cudaError_t e = kernel_setup(k, C::BYTES, kThreads, &nsm, &occ); e != cudaSuccess) return e;
  int64_t grid = static_cast<int64_t>(nsm) * occ;
  if (grid > a.ntiles) grid = a.ntiles;
  if (grid < 1) grid = 1;
  if (info) *info = SolveLaunchInfo{static_cast<int>(grid), kThreads, C::BYTES, occ};
  k<<<static_cast<unsigned>(grid), kThreads, C::BYTES, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

TileCaps solve_caps(int family, int d) {
  auto caps = [](int emax, int Emax, int nmax) { return TileCaps{emax, Emax, nmax}; };
#define TSG_CAPS(DD)                                                                 \
  case DD:                                                                           \
    return family == 0 ? caps(8 * Cfg<DD, 0>::MB, Cfg<DD, 0>::EMAX, Cfg<DD, 0>::NMAX) \
                       : caps(8 * Cfg<DD, 1>::MB, Cfg<DD, 1>::EMAX, Cfg<DD, 1>::NMAX);
  switch (d) {
    TSG_CAPS(2)
    TSG_CAPS(3)
    TSG_CAPS(4)
    TSG_CAPS(5)
    TSG_CAPS(6)
    default:
      return TileCaps{0, 0, 0};
  }
#undef TSG_CAPS
}

cudaError_t launch_solve(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info) {
  if (a.ntiles <= 0) return cudaSuccess;
#define TSG_L(DD)                                                       \
  case DD:                                                              \
    return a.family == 0 ? launch_t<DD, 0>(a, st, info) : launch_t<DD, 1>(a, st, info);
  switch (a.d) {
    TSG_L(2)
    TSG_L(3)
    TSG_L(4)
    TSG_L(5)
    TSG_L(6)
    default:
      return cudaErrorInvalidValue;
  }
#undef TSG_L
}

}  // namespace tsg
