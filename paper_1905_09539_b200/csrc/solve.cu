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

namespace tsg {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxCells = 32;  // Schur cells per mode inside one tile

template <int D, int FAM>
struct Cfg {
  static constexpr int EMAX = (D == 2) ? 1024 : (FAM == 0 ? 4096 : 2048);
  static constexpr int MB = (D == 2) ? 4 : (D == 3 ? 2 : 1);  // e_m <= 8*MB
  static constexpr int NBW = (D == 2) ? 1 : (D == 3 ? 4 : (D == 4 ? 8 : 16));
  static constexpr int NMAX = 64 * NBW;                         // cross-section cap
  static constexpr int KC = (D == 2) ? 16 : (D <= 4 ? 8 : 4);   // K rows per chunk
  static constexpr int LDB = NMAX + 4;                          // == 4 (mod 16)
  static constexpr int MPAD = 8 * MB;
  static constexpr int LDA = MPAD + 4;
  static constexpr int NWB = FAM == 0 ? 0 : D - 1;              // W buffers in smem
  static constexpr int UMAX = D > 5 ? (1 << (D - 5)) : 1;       // unknowns per lane
  static constexpr int HMAX = D * kMaxCells;
  static constexpr int STAGE_B = KC * LDB;
  static constexpr int STAGE_A = KC * LDA;
  static constexpr int DBLK = MPAD * MPAD;                      // diag block per mode
  // shared memory carve-up (doubles, then ints)
  static constexpr int OFF_ACC = 0;
  static constexpr int OFF_W = OFF_ACC + EMAX;
  static constexpr int OFF_B = OFF_W + NWB * EMAX;
  static constexpr int OFF_A = OFF_B + 2 * STAGE_B;
  static constexpr int OFF_D = OFF_A + 2 * STAGE_A;
  static constexpr int NDBLK = FAM == 0 ? D : D + 1;            // + Tc block for gsylv
  static constexpr int OFF_CS = OFF_D + NDBLK * DBLK;           // int64 csoff[NMAX]
  static constexpr int DOUBLES = OFF_CS + NMAX;
  static constexpr int BYTES = DOUBLES * 8 + EMAX * 2 /*cell list u16*/;
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
  int hoff[Cfg<8, 0>::HMAX + 2];
  int cursor[Cfg<8, 0>::HMAX + 2];
};

struct Cplx {
  double re, im;
};
TSG_DEVINL Cplx cmul(Cplx a, Cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
TSG_DEVINL Cplx cadd(Cplx a, Cplx b) { return {a.re + b.re, a.im + b.im}; }
TSG_DEVINL Cplx cdiv(Cplx a, Cplx b) {
  // Smith's algorithm.
  if (fabs(b.re) >= fabs(b.im)) {
    const double r = b.im / b.re, den = b.re + b.im * r;
    return {(a.re + a.im * r) / den, (a.im - a.re * r) / den};
  }
  const double r = b.re / b.im, den = b.re * r + b.im;
  return {(a.re * r + a.im) / den, (a.im * r - a.re) / den};
}

// ---------------------------------------------------------------------------
// Left-looking update pass:  dst -= sum_j  coef_j[rows t_m, later] x_m src_j
// over every tile s later than t along mode m, on DMMA.  The accumulator
// (dst restricted to the tile, M = e_m rows x N = E/e_m cross-section columns)
// stays in registers for the whole pass.
// ---------------------------------------------------------------------------
template <int D, int FAM>
TSG_DEVINL void update_pass(const SolveArgs& a, const TileGeom& tg, double* smem, double* dst,
                            int m, const double* coef0, const double* src0,
                            const double* coef1, const double* src1, int nsrc,
                            double sign) {
  using C = Cfg<D, FAM>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int tm = tg.tco[m];
  const int pm_tiles = a.ntiles_mode[m];
  if (tm + 1 >= pm_tiles) return;  // no later tiles along m (uniform)

  const int em = tg.ext[m];
  const int P = tg.tstride[m];
  const int N = tg.E / em;
  const int NB = (N + 7) >> 3;
  const int MBv = (em + 7) >> 3;
  const int nm = a.dims[m];
  const int64_t sm_stride = a.stride[m];
  int64_t* csoff = reinterpret_cast<int64_t*>(smem + C::OFF_CS);
  double* sB = smem + C::OFF_B;
  double* sA = smem + C::OFF_A;

  // Cross-section offsets (modes != m, mode 0 fastest) of the tile.
  for (int n = tid; n < N; n += kThreads) {
    int rem = n;
    int64_t off = 0;
#pragma unroll
    for (int v = 0; v < D; ++v) {
      if (v == m) continue;
      const int iv = rem % tg.ext[v];
      rem /= tg.ext[v];
      off += static_cast<int64_t>(tg.start[v] + iv) * a.stride[v];
    }
    csoff[n] = off;
  }
  __syncthreads();

  // Load accumulators (C = dst restricted to rows i < em, cols n < N).
  double c[C::MB][C::NBW][2];
#pragma unroll
  for (int ib = 0; ib < C::MB; ++ib)
#pragma unroll
    for (int jj = 0; jj < C::NBW; ++jj)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = ib * 8 + gq, n = (warp + kWarps * jj) * 8 + 2 * tq + h;
        double v = 0.0;
        if (ib < MBv && i < em && n < N) {
          const int q = n / P, p = n - q * P;
          v = dst[p + i * P + q * P * em];
        }
        c[ib][jj][h] = v;
      }

  // Chunk sequence: s from farthest to nearest, each source, K rows by KC.
  struct Chunk {
    int s, j, k0, kv;
  };
  auto first_chunk = [&](Chunk& ch) {
    ch.s = pm_tiles - 1;
    ch.j = 0;
    ch.k0 = 0;
    const int ext_s = a.bnd[m][ch.s + 1] - a.bnd[m][ch.s];
    ch.kv = min(C::KC, ext_s);
  };
  auto next_chunk = [&](Chunk& ch) -> bool {
    const int ext_s = a.bnd[m][ch.s + 1] - a.bnd[m][ch.s];
    ch.k0 += C::KC;
    if (ch.k0 >= ext_s) {
      ch.k0 = 0;
      if (++ch.j >= nsrc) {
        ch.j = 0;
        if (--ch.s <= tm) return false;
      }
    }
    const int ext2 = a.bnd[m][ch.s + 1] - a.bnd[m][ch.s];
    ch.kv = min(C::KC, ext2 - ch.k0);
    return true;
  };
  // Neighbour tile id along m at index s.
  auto nb_tile = [&](int s) -> int64_t {
    int64_t mul = 1;
    for (int v = 0; v < m; ++v) mul *= a.ntiles_mode[v];
    return tg.lt + static_cast<int64_t>(s - tm) * mul;
  };
  auto issue = [&](const Chunk& ch, int buf) {
    const double* coef = ch.j == 0 ? coef0 : coef1;
    const double* src = ch.j == 0 ? src0 : src1;
    const int col0 = a.bnd[m][ch.s] + ch.k0;
    const int row0 = tg.start[m];
    double* A = sA + buf * C::STAGE_A;
    double* B = sB + buf * C::STAGE_B;
    // A chunk: A[k][i] = coef[(row0+i) + (col0+k)*nm]
    for (int e = tid; e < C::KC * C::MPAD; e += kThreads) {
      const int k = e / C::MPAD, i = e - k * C::MPAD;
      const bool ok = (i < em) && (k < ch.kv);
      cp_async8(A + k * C::LDA + i,
                ok ? coef + (row0 + i) + static_cast<int64_t>(col0 + k) * nm : coef, ok ? 8 : 0);
    }
    const int NP = NB * 8;
    if (m == 0) {
      // fibres contiguous along k
      for (int e = tid; e < C::KC * NP; e += kThreads) {
        const int n = e / C::KC, k = e - n * C::KC;
        const bool ok = (k < ch.kv) && (n < N);
        cp_async8(B + k * C::LDB + n,
                  ok ? src + csoff[n] + static_cast<int64_t>(col0 + k) * sm_stride : src,
                  ok ? 8 : 0);
      }
    } else {
      for (int e = tid; e < C::KC * NP; e += kThreads) {
        const int k = e / NP, n = e - k * NP;
        const bool ok = (k < ch.kv) && (n < N);
        cp_async8(B + k * C::LDB + n,
                  ok ? src + csoff[n] + static_cast<int64_t>(col0 + k) * sm_stride : src,
                  ok ? 8 : 0);
      }
    }
  };

  __shared__ int s_waited;
  Chunk cur, nxt;
  first_chunk(cur);
  if (tid == 0) {
    const int* f = a.flags + nb_tile(cur.s);
    while (ld_acquire(f) < a.epoch) __nanosleep(64);
    s_waited = cur.s;
  }
  __syncthreads();
  issue(cur, 0);
  cp_async_commit();
  int buf = 0;
  bool more = true;
  while (more) {
    nxt = cur;
    const bool has_next = next_chunk(nxt);
    if (has_next && tid == 0 && nxt.s != s_waited) {
      const int* f = a.flags + nb_tile(nxt.s);
      while (ld_acquire(f) < a.epoch) __nanosleep(64);
      s_waited = nxt.s;
    }
    __syncthreads();
    if (has_next) issue(nxt, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* A = sA + buf * C::STAGE_A;
    const double* B = sB + buf * C::STAGE_B;
#pragma unroll
    for (int k4 = 0; k4 < C::KC; k4 += 4) {
      double af[C::MB], bf[C::NBW];
#pragma unroll
      for (int ib = 0; ib < C::MB; ++ib) af[ib] = sign * A[(k4 + tq) * C::LDA + ib * 8 + gq];
#pragma unroll
      for (int jj = 0; jj < C::NBW; ++jj) {
        const int jb = warp + kWarps * jj;
        bf[jj] = (jb < NB) ? B[(k4 + tq) * C::LDB + jb * 8 + gq] : 0.0;
      }
#pragma unroll
      for (int ib = 0; ib < C::MB; ++ib) {
        if (ib >= MBv) continue;
#pragma unroll
        for (int jj = 0; jj < C::NBW; ++jj) {
          if (warp + kWarps * jj >= NB) continue;
          dmma(c[ib][jj][0], c[ib][jj][1], af[ib], bf[jj]);
        }
      }
    }
    cur = nxt;
    more = has_next;
    buf ^= 1;
  }
  cp_async_wait_all();

  // Store accumulators back.
#pragma unroll
  for (int ib = 0; ib < C::MB; ++ib)
#pragma unroll
    for (int jj = 0; jj < C::NBW; ++jj)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = ib * 8 + gq, n = (warp + kWarps * jj) * 8 + 2 * tq + h;
        if (ib < MBv && i < em && n < N) {
          const int q = n / P, p = n - q * P;
          dst[p + i * P + q * P * em] = c[ib][jj][h];
        }
      }
  __syncthreads();
}

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

// Per-lane view of the cell currently handled by this lane group.
template <int D>
struct CellView {
  int c[D];         // cell coordinates
  int valid;        // group has a cell this round
};

template <int D, int FAM>
__global__ void __launch_bounds__(kThreads, 1) solve_kernel(SolveArgs a) {
  using C = Cfg<D, FAM>;
  extern __shared__ __align__(16) double smem[];
  __shared__ TileGeom tg;
  __shared__ int s_tile;
  double* acc = smem + C::OFF_ACC;
  double* wbuf = smem + C::OFF_W;  // wbuf + (m-1)*EMAX for m = 1..D-1 (gsylv)
  double* dblk = smem + C::OFF_D;  // D diag blocks (+ Tc block for gsylv)
  unsigned short* clist = reinterpret_cast<unsigned short*>(smem + C::DOUBLES);
  const int tid = threadIdx.x, lane = tid & 31;

  for (;;) {
    if (tid == 0) s_tile = atomicAdd(a.counter, 1);
    __syncthreads();
    const int qi = s_tile;
    if (qi >= a.ntiles) break;

    // ---- tile geometry + Schur cells (thread 0) ---------------------------
    if (tid == 0) {
      const int64_t lt = a.order[qi];
      tg.lt = lt;
      int64_t rem = lt, gb = 0;
      int E = 1, H = 0, ncell = 1, kp = 0;
      for (int m = 0; m < D; ++m) {
        const int tm = static_cast<int>(rem % a.ntiles_mode[m]);
        rem /= a.ntiles_mode[m];
        tg.tco[m] = tm;
        const int st = a.bnd[m][tm];
        const int ex = a.bnd[m][tm + 1] - st;
        tg.start[m] = st;
        tg.ext[m] = ex;
        tg.tstride[m] = E;
        E *= ex;
        gb += static_cast<int64_t>(st) * a.stride[m];
        int nc = 0;
        bool pair = false;
        for (int r = 0; r < ex;) {
          const int sz = (a.blk[m][st + r] == 1) ? 2 : 1;
          tg.cs[m][nc] = static_cast<unsigned char>(r);
          tg.cz[m][nc] = static_cast<unsigned char>(sz);
          pair |= (sz == 2);
          ++nc;
          r += sz;
        }
        tg.nc[m] = nc;
        ncell *= nc;
        H += nc - 1;
        tg.pidx[m] = pair ? kp : -1;
        if (pair) tg.pm[kp++] = m;
      }
      tg.E = E;
      tg.gbase = gb;
      tg.ncell = ncell;
      tg.H = H;
      tg.kp = kp;
      for (int h = 0; h <= H + 1; ++h) tg.hoff[h] = 0;
    }
    __syncthreads();
    const int E = tg.E;

    // ---- gather B~_t, stage diagonal blocks, zero W partials ---------------
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
    // Hyperplane histogram of the cells.
    for (int cid = tid; cid < tg.ncell; cid += kThreads) {
      int rem = cid, h = 0;
#pragma unroll
      for (int v = 0; v < D; ++v) {
        h += rem % tg.nc[v];
        rem /= tg.nc[v];
      }
      atomicAdd(&tg.hoff[h + 1], 1);
    }
    cp_async_wait_all();
    __syncthreads();
    if (tid == 0) {
      for (int h = 0; h <= tg.H; ++h) {
        tg.hoff[h + 1] += tg.hoff[h];
        tg.cursor[h] = tg.hoff[h];
      }
    }
    __syncthreads();
    for (int cid = tid; cid < tg.ncell; cid += kThreads) {
      int rem = cid, h = 0;
#pragma unroll
      for (int v = 0; v < D; ++v) {
        h += rem % tg.nc[v];
        rem /= tg.nc[v];
      }
      clist[atomicAdd(&tg.cursor[h], 1)] = static_cast<unsigned short>(cid);
    }

    // ---- left-looking off-diagonal updates (DMMA) --------------------------
    if (FAM == 0) {
      for (int m = 0; m < D; ++m)
        update_pass<D, FAM>(a, tg, smem, acc, m, a.T[m], a.X, nullptr, nullptr, 1, -1.0);
    } else {
      // mode 0: acc -= S[t0, later] x_0 X  +  Tc[t0, later] x_0 V
      update_pass<D, FAM>(a, tg, smem, acc, 0, a.T[0], a.X, a.Tc, a.W[1], 2, -1.0);
      // tails: W'_m = sum_{later s} A_m[t_m, s] x_m W_{m+1}   (W_D == X)
      for (int m = 1; m < D; ++m)
        update_pass<D, FAM>(a, tg, smem, wbuf + (m - 1) * C::EMAX, m, a.T[m],
                            m == D - 1 ? a.X : a.W[m + 1], nullptr, nullptr, 1, 1.0);
    }
    __syncthreads();

    // ---- in-tile wavefront over Schur cells --------------------------------
    {
      const int kp = tg.kp;
      const int LB = kp < 5 ? kp : 5;
      const int G = 1 << LB;
      const int NG = kThreads / G;
      const int gid = tid / G, lig = tid & (G - 1);
      const int U = 1 << (kp > 5 ? kp - 5 : 0);
      for (int h = tg.H; h >= 0; --h) {
        const int cbeg = tg.hoff[h], ccount = tg.hoff[h + 1] - cbeg;
        const int rounds = (ccount + NG - 1) / NG;
        for (int rd = 0; rd < rounds; ++rd) {
          const int slot = rd * NG + gid;
          const bool gvalid = slot < ccount;
          int c[D];
          {
            int rem = gvalid ? clist[cbeg + slot] : 0;
#pragma unroll
            for (int v = 0; v < D; ++v) {
              c[v] = rem % tg.nc[v];
              rem /= tg.nc[v];
            }
          }
          // Unknowns of this lane.
          int off[C::UMAX];
          bool present[C::UMAX];
          int loc[C::UMAX][D];  // tile-local coordinates
#pragma unroll
          for (int u = 0; u < C::UMAX; ++u) {
            const int bits = lig | (u << LB);
            bool pres = gvalid && (u < U);
            int o = 0;
#pragma unroll
            for (int v = 0; v < D; ++v) {
              const int b = tg.pidx[v] >= 0 ? (bits >> tg.pidx[v]) & 1 : 0;
              const int cz = tg.cz[v][c[v]];
              if (b && cz == 1) pres = false;
              const int iv = tg.cs[v][c[v]] + (cz == 2 ? b : 0);
              loc[u][v] = iv;
              o += iv * tg.tstride[v];
            }
            present[u] = pres;
            off[u] = o;
          }
          // Eigen data of each pair mode's block for this cell.
          // Residuals (left-looking in-tile dots) -------------------------
          double r[C::UMAX];
          if (FAM == 0) {
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) {
              double s = 0.0;
              if (present[u]) {
                s = acc[off[u]];
#pragma unroll
                for (int v = 0; v < D; ++v) {
                  const int em = tg.ext[v];
                  const int iv = loc[u][v];
                  const int jend = tg.cs[v][c[v]] + tg.cz[v][c[v]];
                  const double* Dv = dblk + v * C::DBLK;
                  const int ts = tg.tstride[v];
                  for (int j = jend; j < em; ++j) s -= Dv[iv + j * em] * acc[off[u] + (j - iv) * ts];
                }
              }
              r[u] = s;
            }
          }
          // gsylv: tail partials P_m, chain R, mode-0 residual.
          double P[C::UMAX][D];
          if (FAM == 1) {
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) {
#pragma unroll
              for (int v = 1; v < D; ++v) {
                double s = 0.0;
                if (present[u]) {
                  s = wbuf[(v - 1) * C::EMAX + off[u]];
                  const double* srcb = (v == D - 1) ? acc : wbuf + v * C::EMAX;
                  const int em = tg.ext[v];
                  const int iv = loc[u][v];
                  const int jend = tg.cs[v][c[v]] + tg.cz[v][c[v]];
                  const double* Dv = dblk + v * C::DBLK;
                  const int ts = tg.tstride[v];
                  for (int j = jend; j < em; ++j)
                    s += Dv[iv + j * em] * srcb[off[u] + (j - iv) * ts];
                }
                P[u][v] = s;
              }
            }
          }
          // helpers -----------------------------------------------------------
          auto bit_of = [&](int u, int j) { return ((lig | (u << LB)) >> j) & 1; };
          // y <- A_v,cc x_v y with the cell's diagonal block of `blk` (tile-local,
          // ld e_v).  Shuffles are issued whenever v is a pair mode of the tile
          // (tile-uniform), so lane groups holding 1x1 cells stay converged.
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
                for (int u = 0; u < C::UMAX; ++u) {
                  const int b = bit_of(u, j);
                  y[u] = b == 0 ? a00 * y[u] + a01 * py[u] : a10 * py[u] + a11 * y[u];
                }
                return;
              }
            }
            const double d0 = blk[i0 + i0 * em];
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) y[u] *= d0;
          };
          // Complex butterfly with eigen data (inv: V^{-1}, else V) of pair mode v.
          auto eig_apply = [&](Cplx (&z)[C::UMAX], int v, bool inv) {
            const int j = tg.pidx[v];
            if (j < 0) return;
            Cplx pz[C::UMAX];
            partner_c<C::UMAX>(z, pz, j, LB);
            if (tg.cz[v][c[v]] != 2) return;
            const double* ed = a.eig[v] + static_cast<int64_t>(tg.start[v] + tg.cs[v][c[v]]) * kEigStride;
            const double* M = ed + (inv ? 4 : 12);
            const Cplx m00{M[0], M[1]}, m01{M[2], M[3]}, m10{M[4], M[5]}, m11{M[6], M[7]};
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) {
              const int b = bit_of(u, j);
              z[u] = b == 0 ? cadd(cmul(m00, z[u]), cmul(m01, pz[u]))
                            : cadd(cmul(m10, pz[u]), cmul(m11, z[u]));
            }
          };
          auto lam_of = [&](int u, int v) -> Cplx {
            // eigenvalue of mode v's cell block for this unknown's bit
            const int i0 = tg.cs[v][c[v]];
            if (tg.cz[v][c[v]] == 2) {
              const int j = tg.pidx[v];
              const double* ed = a.eig[v] + static_cast<int64_t>(tg.start[v] + i0) * kEigStride;
              const int b = bit_of(u, j);
              return Cplx{ed[2 * b], ed[2 * b + 1]};
            }
            return Cplx{dblk[v * C::DBLK + i0 + i0 * tg.ext[v]], 0.0};
          };

          // Closed-form cell solve: y = cellop^{-1} rhs (real in, real out).
          bool singular = false;
          auto cell_solve = [&](const double (&rhs)[C::UMAX], double (&y)[C::UMAX]) {
            Cplx z[C::UMAX];
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) z[u] = Cplx{rhs[u], 0.0};
            const int v_first = (FAM == 0) ? 0 : 1;
            for (int v = v_first; v < D; ++v) eig_apply(z, v, true);
            if (FAM == 0) {
#pragma unroll
              for (int u = 0; u < C::UMAX; ++u) {
                Cplx mu{0.0, 0.0};
                for (int v = 0; v < D; ++v) mu = cadd(mu, lam_of(u, v));
                if (fabs(mu.re) + fabs(mu.im) <= a.tiny) {
                  singular = singular || present[u];
                  mu = Cplx{1.0, 0.0};
                }
                z[u] = cdiv(z[u], mu);
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
                  const int b = bit_of(u, j0);
                  // x0 = (m11 r0 - m01 r1)/det ; x1 = (m00 r1 - m10 r0)/det
                  const Cplx r0 = b == 0 ? z[u] : pz[u];
                  const Cplx r1 = b == 0 ? pz[u] : z[u];
                  const Cplx num = b == 0 ? cadd(cmul(m11, r0), cmul(Cplx{-m01.re, -m01.im}, r1))
                                          : cadd(cmul(m00, r1), cmul(Cplx{-m10.re, -m10.im}, r0));
                  z[u] = cdiv(num, det);
                }
              }
            }
            for (int v = D - 1; v >= v_first; --v) eig_apply(z, v, false);
#pragma unroll
            for (int u = 0; u < C::UMAX; ++u) y[u] = present[u] ? z[u].re : 0.0;
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
                s = acc[off[u]] - R[u];
                const int e0 = tg.ext[0];
                const int i0 = loc[u][0];
                const int jend = tg.cs[0][c[0]] + tg.cz[0][c[0]];
                const double* Sb = dblk;
                const double* Tb = dblk + D * C::DBLK;
                const double* Vb = wbuf;  // W_1 == V
                for (int j = jend; j < e0; ++j) {
                  const int o2 = off[u] + (j - i0);
                  s -= Sb[i0 + j * e0] * acc[o2] + Tb[i0 + j * e0] * Vb[o2];
                }
              }
              r[u] = s;
            }
          }

          double y[C::UMAX], res[C::UMAX], dy[C::UMAX];
          cell_solve(r, y);
          cell_op(y, res);
#pragma unroll
          for (int u = 0; u < C::UMAX; ++u) res[u] = present[u] ? r[u] - res[u] : 0.0;
          cell_solve(res, dy);
#pragma unroll
          for (int u = 0; u < C::UMAX; ++u) y[u] += dy[u];

          if (singular && gvalid) atomicMin(a.status, static_cast<int>(tg.lt < 0x7f7f7f7e ? tg.lt : 0x7f7f7f7e));
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
  (void)lane;
}

template <int D, int FAM>
cudaError_t launch_t(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info) {
  using C = Cfg<D, FAM>;
  auto k = solve_kernel<D, FAM>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::BYTES);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, C::BYTES);
  if (e != cudaSuccess) return e;
  if (occ < 1) occ = 1;
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
