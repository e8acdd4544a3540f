// Fast path of the reduced Laplace-like solve (family 0): persistent
// dataflow over small tiles (8^3 class) with many CTAs per SM.
//
// Same schedule as solve.cu (tiles in topological hyperplane order through an
// atomic queue, left-looking DMMA updates from later tiles, release flags),
// but the in-tile base case works in the eigenbasis of the tile's diagonal
// Schur blocks:
//   * every 1x1/2x2 diagonal block of T_m is P diag(l0, l1) P^{-1} with
//     P = W E (W the real normal-form similarity, E the fixed butterfly
//     [[1, 1], [i, -i]]), so one block-diagonal transform per mode turns the
//     tile's Kronecker-sum operator sum_m I (x) That_m (x) I into an upper
//     TRIANGULAR complex operator with diagonal mu(u) = sum_m lambda_m(i_m);
//   * the wavefront over Schur-cell hyperplanes then solves every unknown on
//     the hyperplane independently:
//        xhat(u) = (rhat(u) - sum_m sum_{j beyond u's cell} That_m[i_m, j] xhat(u|m->j)) / mu(u)
//     with no intra-cell coupling (no shuffles, no lane groups);
//   * the tile is transformed back with P along each mode (real part).
// Unknowns are pre-sorted by cell hyperplane once per tile, so every
// wavefront step is one pass of independent lanes plus one barrier.
// Reference path replaced: lap_rec / lap_base / block_back_substitution
// (laplace.hpp:99-153, kernels.hpp:179-261).
#include <climits>
#include <cstdint>

#include "common.cuh"
#include "solve.h"
#include "solve_common.cuh"
#include "util.h"

namespace tsg {
namespace {

template <int D>
struct LapCfg {
  static constexpr int THREADS = 128;
  static constexpr int EMAX = 512;
  static constexpr int MB = (D == 2) ? 4 : 1;  // e_m <= 8*MB
  static constexpr int NBW = (D == 2) ? 1 : (D == 3 ? 2 : (D == 4 ? 4 : 8));
  static constexpr int NMAX = 8 * (THREADS / 32) * NBW;  // cross-section cap
  static constexpr int KC = (D <= 3) ? 16 : 8;
  static constexpr int NSTAGE = 3;
  static constexpr int LDB = NMAX + 4;  // == 4 (mod 16)
  static constexpr int MPAD = 8 * MB;
  static constexpr int LDA = MPAD + 4;
  static constexpr int STAGE_B = KC * LDB;
  static constexpr int STAGE_A = KC * LDA;
  static constexpr int EM = MPAD;  // max tile extent per mode
  // shared memory (doubles)
  static constexpr int OFF_ACC = 0;
  static constexpr int OFF_XR = OFF_ACC + EMAX;
  static constexpr int OFF_XI = OFF_XR + EMAX;
  static constexpr int OFF_B = OFF_XI + EMAX;
  static constexpr int OFF_A = OFF_B + NSTAGE * STAGE_B;
  static constexpr int OFF_DH = OFF_A + NSTAGE * STAGE_A;      // That_m (re, im): 2*EM*EM per mode
  static constexpr int OFF_LAM = OFF_DH + D * 2 * EM * EM;      // lambda_m (re, im): 2*EM per mode
  static constexpr int OFF_PD = OFF_LAM + D * 2 * EM;          // P/Pinv data of tile rows
  static constexpr int OFF_DB = OFF_PD + D * EM * kPStride;    // real diag blocks (EM*EM per mode)
  static constexpr int OFF_CS = OFF_DB + D * EM * EM;          // int64 csoff[NMAX]
  static constexpr int DOUBLES = OFF_CS + NMAX;
  static constexpr int BYTES = DOUBLES * 8 + EMAX * 4 /* sorted unknowns */;
};

struct LapGeom {
  int64_t lt;
  int64_t gbase;
  int start[kMaxOrder], ext[kMaxOrder], tco[kMaxOrder], tstride[kMaxOrder];
  int E, H, kp;
  int nc[kMaxOrder];
  unsigned char cs[kMaxOrder][kMaxCells], cz[kMaxOrder][kMaxCells];
  unsigned char cellof[kMaxOrder][32];  // row (tile-local) -> cell index
  unsigned char cend[kMaxOrder][32];    // row -> first row after its cell
  int hoff[kMaxOrder * kMaxCells + 2];
  int cursor[kMaxOrder * kMaxCells + 2];
};

template <int D>
__global__ void __launch_bounds__(LapCfg<D>::THREADS) solve_lap_kernel(SolveArgs a) {
  using C = LapCfg<D>;
  constexpr int T = C::THREADS;
  constexpr int EM = C::EM;
  extern __shared__ __align__(16) double smem[];
  __shared__ LapGeom tg;
  __shared__ int s_tile;
  double* acc = smem + C::OFF_ACC;
  double* xr = smem + C::OFF_XR;
  double* xi = smem + C::OFF_XI;
  double* dh = smem + C::OFF_DH;
  double* lam = smem + C::OFF_LAM;
  double* pd = smem + C::OFF_PD;
  double* db = smem + C::OFF_DB;
  unsigned* ulist = reinterpret_cast<unsigned*>(smem + C::DOUBLES);
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

    // ---- geometry: host-packed tile coordinates + per-mode tables ----------
    if (tid < D) {
      const unsigned long long pk = a.ocoord[qi];
      const int tm = static_cast<int>((pk >> (10 * tid)) & 1023);
      const TileMode& src = a.tmode[tid][tm];
      tg.tco[tid] = tm;
      tg.start[tid] = src.start;
      tg.ext[tid] = src.ext;
      tg.nc[tid] = src.nc;
      for (int k = 0; k < src.nc; ++k) {
        const int s0 = src.cs[k], sz = src.cz[k];
        tg.cs[tid][k] = static_cast<unsigned char>(s0);
        tg.cz[tid][k] = static_cast<unsigned char>(sz);
        for (int r = s0; r < s0 + sz; ++r) {
          tg.cellof[tid][r] = static_cast<unsigned char>(k);
          tg.cend[tid][r] = static_cast<unsigned char>(s0 + sz);
        }
      }
      if (tid == 0) {
        tg.lt = a.order[qi];
        tg.kp = 0;
      }
    }
    __syncthreads();
    if (tid == 0) {
      int64_t gb = 0;
      int E = 1, H = 0, kp = 0;
      for (int m = 0; m < D; ++m) {
        tg.tstride[m] = E;
        E *= tg.ext[m];
        gb += static_cast<int64_t>(tg.start[m]) * a.stride[m];
        H += tg.nc[m] - 1;
        bool pair = false;
        for (int k = 0; k < tg.nc[m]; ++k) pair |= tg.cz[m][k] == 2;
        kp += pair ? 1 : 0;
      }
      tg.E = E;
      tg.gbase = gb;
      tg.H = H;
      tg.kp = kp;
      for (int h = 0; h <= H + 1; ++h) tg.hoff[h] = 0;
    }
    __syncthreads();
    const int E = tg.E;

    // ---- gather B~_t; stage diag blocks + P data; hyperplane histogram -------
    for (int l = tid; l < E; l += T) {
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
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int em = tg.ext[m], st = tg.start[m], nm = a.dims[m];
      for (int e = tid; e < em * em; e += T) {
        const int i = e % em, j = e / em;
        db[m * EM * EM + i + j * EM] = a.T[m][(st + i) + static_cast<int64_t>(st + j) * nm];
      }
      for (int e = tid; e < em * kPStride; e += T)
        pd[m * EM * kPStride + e] = a.pdat[m][static_cast<int64_t>(st) * kPStride + e];
    }
    for (int l = tid; l < E; l += T) {
      int rem = l, h = 0;
#pragma unroll
      for (int v = 0; v < D; ++v) {
        h += tg.cellof[v][rem % tg.ext[v]];
        rem /= tg.ext[v];
      }
      atomicAdd(&tg.hoff[h + 1], 1);
    }
    __syncthreads();
    if (tid == 0) {
      for (int h = 0; h <= tg.H; ++h) {
        tg.hoff[h + 1] += tg.hoff[h];
        tg.cursor[h] = tg.hoff[h];
      }
    }
    __syncthreads();
    // sorted unknowns: packed tile-local coordinates (5 bits per mode)
    for (int l = tid; l < E; l += T) {
      int rem = l, h = 0;
      unsigned pk = 0;
#pragma unroll
      for (int v = 0; v < D; ++v) {
        const int iv = rem % tg.ext[v];
        rem /= tg.ext[v];
        h += tg.cellof[v][iv];
        pk |= static_cast<unsigned>(iv) << (5 * v);
      }
      ulist[atomicAdd(&tg.cursor[h], 1)] = pk;
    }
    // That_m = Pinv_blk(i) D_m P_blk(j) on the strictly-later-cell part, and
    // lambda_m (the diagonal).  P data row layout (kPStride doubles at a
    // block's first row): l0, l1 (complex), P (2x2 complex, row-major),
    // Pinv (2x2 complex, row-major).
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int em = tg.ext[m];
      const double* dm = db + m * EM * EM;
      const double* pm = pd + m * EM * kPStride;
      for (int e = tid; e < em * em; e += T) {
        const int i = e % em, j = e / em;
        double re = 0.0, im = 0.0;
        if (j >= tg.cend[m][i]) {
          const int I0 = tg.cs[m][tg.cellof[m][i]], Iz = tg.cz[m][tg.cellof[m][i]];
          const int J0 = tg.cs[m][tg.cellof[m][j]], Jz = tg.cz[m][tg.cellof[m][j]];
          const double* pi = pm + I0 * kPStride + 12;  // Pinv of block(i)
          const double* pj = pm + J0 * kPStride + 4;   // P of block(j)
          for (int aa = 0; aa < Iz; ++aa) {
            // w = Pinv[i-I0][aa] (complex) or 1 for a 1x1 block
            const double wr = Iz == 2 ? pi[((i - I0) * 2 + aa) * 2] : 1.0;
            const double wi = Iz == 2 ? pi[((i - I0) * 2 + aa) * 2 + 1] : 0.0;
            for (int bb = 0; bb < Jz; ++bb) {
              const double d = dm[(I0 + aa) + (J0 + bb) * EM];
              const double vr = Jz == 2 ? pj[(bb * 2 + (j - J0)) * 2] : 1.0;
              const double vi = Jz == 2 ? pj[(bb * 2 + (j - J0)) * 2 + 1] : 0.0;
              // w * d * v
              re += d * (wr * vr - wi * vi);
              im += d * (wr * vi + wi * vr);
            }
          }
        }
        dh[m * 2 * EM * EM + i + j * EM] = re;
        dh[m * 2 * EM * EM + EM * EM + i + j * EM] = im;
      }
      for (int i = tid; i < em; i += T) {
        const int I0 = tg.cs[m][tg.cellof[m][i]];
        const double* p = pm + I0 * kPStride + (i - I0) * 2;  // l0 or l1
        lam[m * 2 * EM + i] = p[0];
        lam[m * 2 * EM + EM + i] = p[1];
      }
    }
    cp_async_wait_all();
    __syncthreads();
    mark(1);

    // ---- left-looking off-diagonal updates (DMMA): far tiles, then near ------
    for (int part = 0; part < 2; ++part) {
      int64_t mul = 1;
#pragma unroll 1
      for (int m = 0; m < D; ++m) {
        const int tm = tg.tco[m], pmt = a.ntiles_mode[m];
        const int* bm = a.bnd[m];
        int k_lo = 0, k_hi = 0, wt = -1;
        if (part == 0 && tm + 2 < pmt) {
          k_lo = bm[tm + 2];
          k_hi = a.dims[m];
          wt = tm + 2;
        } else if (part == 1 && tm + 1 < pmt) {
          k_lo = bm[tm + 1];
          k_hi = bm[tm + 2];
          wt = tm + 1;
        }
        if (wt >= 0 && !(a.dbg & 4))
          update_pass<D, C>(a, tg, smem, acc, m, k_lo, k_hi, tg.lt + (wt - tm) * mul, a.T[m], a.X,
                            nullptr, nullptr, 1, -1.0);
        mul *= pmt;
      }
    }

    mark(2);
    // ---- into the eigenbasis: x = acc x_m Pinv_m  (pair modes only) ----------
    const bool cplx = tg.kp > 0;
    for (int l = tid; l < E; l += T) {
      xr[l] = acc[l];
      xi[l] = 0.0;
    }
    __syncthreads();
    if (cplx) {
#pragma unroll 1
      for (int m = 0; m < D; ++m) {
        const int em = tg.ext[m], ts = tg.tstride[m];
        const double* pm = pd + m * EM * kPStride;
        // one thread per (row pair start, cross-section) position
        for (int l = tid; l < E; l += T) {
          const int i = (l / ts) % em;
          const int ci = tg.cellof[m][i];
          if (tg.cz[m][ci] != 2 || tg.cs[m][ci] != i) continue;
          const double* pi = pm + i * kPStride + 12;
          const int l2 = l + ts;
          const double ar = xr[l], ai = xi[l], br = xr[l2], bi = xi[l2];
          // y0 = Pinv00 a + Pinv01 b ; y1 = Pinv10 a + Pinv11 b
          xr[l] = pi[0] * ar - pi[1] * ai + pi[2] * br - pi[3] * bi;
          xi[l] = pi[0] * ai + pi[1] * ar + pi[2] * bi + pi[3] * br;
          xr[l2] = pi[4] * ar - pi[5] * ai + pi[6] * br - pi[7] * bi;
          xi[l2] = pi[4] * ai + pi[5] * ar + pi[6] * bi + pi[7] * br;
        }
        __syncthreads();
      }
    }

    mark(3);
    // ---- wavefront over cell hyperplanes (independent unknowns) -------------
    bool singular = false;
#pragma unroll 1
    for (int h = (a.dbg & 1) ? -1 : tg.H; h >= 0; --h) {
      const int beg = tg.hoff[h], end = tg.hoff[h + 1];
      for (int idx = beg + tid; idx < end; idx += T) {
        const unsigned pk = ulist[idx];
        int iv[D], off = 0;
#pragma unroll
        for (int v = 0; v < D; ++v) {
          iv[v] = (pk >> (5 * v)) & 31;
          off += iv[v] * tg.tstride[v];
        }
        double sr[D], si[D];
        double mur = 0.0, mui = 0.0;
#pragma unroll
        for (int v = 0; v < D; ++v) {
          const int em = tg.ext[v], ts = tg.tstride[v];
          const int i = iv[v];
          const double* dr = dh + v * 2 * EM * EM + i;
          const double* di = dr + EM * EM;
          const double* pr = xr + off - i * ts;
          const double* pim = xi + off - i * ts;
          double ar = 0.0, ai = 0.0;
          if (cplx) {
            for (int j = tg.cend[v][i]; j < em; ++j) {
              const double cr = dr[j * EM], ci = di[j * EM];
              const double yr = pr[j * ts], yi = pim[j * ts];
              ar = fma(cr, yr, ar);
              ar = fma(-ci, yi, ar);
              ai = fma(cr, yi, ai);
              ai = fma(ci, yr, ai);
            }
          } else {
            for (int j = tg.cend[v][i]; j < em; ++j) ar = fma(dr[j * EM], pr[j * ts], ar);
          }
          sr[v] = ar;
          si[v] = ai;
          mur += lam[v * 2 * EM + i];
          mui += lam[v * 2 * EM + EM + i];
        }
        double rr = xr[off], ri = xi[off];
#pragma unroll
        for (int v = 0; v < D; ++v) {
          rr -= sr[v];
          ri -= si[v];
        }
        const double den = mur * mur + mui * mui;
        if (!(den > a.tiny * a.tiny)) {
          singular = true;
          xr[off] = 0.0;
          xi[off] = 0.0;
        } else {
          const double inv = 1.0 / den;
          xr[off] = (rr * mur + ri * mui) * inv;
          xi[off] = (ri * mur - rr * mui) * inv;
        }
      }
      __syncthreads();
    }
    if (singular)
      atomicMin(a.status, static_cast<int>(tg.lt < 0x7f7f7f7e ? tg.lt : 0x7f7f7f7e));

    mark(4);
    // ---- back to the Schur basis: X = xhat x_m P_m, real part ---------------
    if (cplx) {
#pragma unroll 1
      for (int m = 0; m < D; ++m) {
        const int em = tg.ext[m], ts = tg.tstride[m];
        const double* pm = pd + m * EM * kPStride;
        for (int l = tid; l < E; l += T) {
          const int i = (l / ts) % em;
          const int ci = tg.cellof[m][i];
          if (tg.cz[m][ci] != 2 || tg.cs[m][ci] != i) continue;
          const double* p = pm + i * kPStride + 4;
          const int l2 = l + ts;
          const double ar = xr[l], ai = xi[l], br = xr[l2], bi = xi[l2];
          xr[l] = p[0] * ar - p[1] * ai + p[2] * br - p[3] * bi;
          xi[l] = p[0] * ai + p[1] * ar + p[2] * bi + p[3] * br;
          xr[l2] = p[4] * ar - p[5] * ai + p[6] * br - p[7] * bi;
          xi[l2] = p[4] * ai + p[5] * ar + p[6] * bi + p[7] * br;
        }
        __syncthreads();
      }
    }

    mark(5);
    // ---- scatter X_t, release -------------------------------------------------
    for (int l = tid; l < E; l += T) {
      int rem = l;
      int64_t off = tg.gbase;
#pragma unroll
      for (int v = 0; v < D; ++v) {
        const int ivv = rem % tg.ext[v];
        rem /= tg.ext[v];
        off += static_cast<int64_t>(ivv) * a.stride[v];
      }
      a.X[off] = xr[l];
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(a.flags + tg.lt, a.epoch);
    }
    mark(6);
    if (a.prof && tid == 0) atomicAdd(a.prof + 8, 1ull);
  }
  if (a.prof && tid == 0)
    for (int k = 0; k < 8; ++k) atomicAdd(a.prof + k, ph[k]);
}

template <int D>
cudaError_t launch_lap_t(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info) {
  using C = LapCfg<D>;
  auto k = solve_lap_kernel<D>;
  int nsm = 0, occ = 0;
  if (cudaError_t e = kernel_setup(k, C::BYTES, C::THREADS, &nsm, &occ); e != cudaSuccess) return e;
  int64_t grid = static_cast<int64_t>(nsm) * occ;
  if (grid > a.ntiles) grid = a.ntiles;
  if (grid < 1) grid = 1;
  if (info) *info = SolveLaunchInfo{static_cast<int>(grid), C::THREADS, C::BYTES, occ};
  k<<<static_cast<unsigned>(grid), C::THREADS, C::BYTES, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

TileCaps solve_lap_caps(int d) {
  switch (d) {
    case 2:
      return TileCaps{8 * LapCfg<2>::MB, LapCfg<2>::EMAX, LapCfg<2>::NMAX};
    case 3:
      return TileCaps{8 * LapCfg<3>::MB, LapCfg<3>::EMAX, LapCfg<3>::NMAX};
    case 4:
      return TileCaps{8 * LapCfg<4>::MB, LapCfg<4>::EMAX, LapCfg<4>::NMAX};
    case 5:
      return TileCaps{8 * LapCfg<5>::MB, LapCfg<5>::EMAX, LapCfg<5>::NMAX};
    case 6:
      return TileCaps{8 * LapCfg<6>::MB, LapCfg<6>::EMAX, LapCfg<6>::NMAX};
    default:
      return TileCaps{0, 0, 0};
  }
}

cudaError_t launch_solve_lap(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info) {
  if (a.ntiles <= 0) return cudaSuccess;
  switch (a.d) {
    case 2:
      return launch_lap_t<2>(a, st, info);
    case 3:
      return launch_lap_t<3>(a, st, info);
    case 4:
      return launch_lap_t<4>(a, st, info);
    case 5:
      return launch_lap_t<5>(a, st, info);
    case 6:
      return launch_lap_t<6>(a, st, info);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace tsg
