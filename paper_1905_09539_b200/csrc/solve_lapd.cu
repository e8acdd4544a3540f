// Higher-order Laplace-like solve (d = 4..6, e.g. C3 = 24^6): the dataflow
// of solve_lap3.cu on small d-dimensional tiles (padded extents 2/4/8,
// at most 512 unknowns), four CTAs of 128 threads per SM.
//
// Per tile:
//   1. gather B~_t (cp.async, padded power-of-two layout) and the complex
//      eigenvector bases of its d diagonal Schur blocks (host tables, the
//      same 8x8 identity-padded V^-1 | V | lambda records as solve_lap3);
//   2. left-looking updates in two passes (tiles >= t+2 first, then the t+1
//      neighbours after their flags): for every mode the tile's cross-section
//      is split over the warps in 8-column blocks and
//        Y(cross, rows) -= X(cross, k) T_m(rows, k)^T
//      runs on DMMA with X as the A operand (so a small tile extent e_m only
//      pads the N side of the 8x8x4 product; each X element is loaded once);
//   3. diagonalised base case: x^ = x x_m V_m^-1 (all modes), divide by
//      sum_m lambda_m, x = x^ x_m V_m, one thread per fibre (P_m <= 8);
//   4. scatter, release.
// Reference: lap_rec / lap_base (laplace.hpp:99-153), the merged-mode base
// case laplace_merged (laplace.hpp:202-244), mode_multiply (laplace.hpp:147).
#include <cstdint>

#include "common.cuh"
#include "solve.h"
#include "util.h"

#ifndef LAPD_PROF
#define LAPD_PROF 0
#endif

namespace tsg {
namespace {

#ifndef LAPD_EP
#define LAPD_EP 512
#endif
constexpr int EP = LAPD_EP, THREADS = EP / 4, WARPS = THREADS / 32;
constexpr int VHS = kVhStride;  // 8x8 complex records (tile_eigvecs<8>)

template <int D>
struct GD {
  int64_t lt, gbase;
  int start[D], ext[D], tco[D];
};

TSG_DEVINL void waitp(const SolveArgs& a, int64_t tile) {
  const int* f = a.flags + tile;
  unsigned ns = 32;
  while (ld_acquire(f) < a.epoch) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
}

// xr -= sum_k X(cross, k) T_m(rows, k) over rows k in [klo, khi) of mode m
// (cross-section of ep >> log2 P_m columns, 8-column blocks dealt to the
// warps, NBMAX blocks per warp and round)
// tile-local offset of the first element of fibre f along mode m: the
// tile index is the concatenation of the modes' bit fields (mode 0 lowest),
// so dropping mode m's field from a fibre index = inserting tlog[m] zero
// bits at tsh[m]
template <int D>
TSG_DEVINL int fibre_lt(const SolveArgs& a, int m, int f) {
  const int sh = a.tsh[m];
  return (f & ((1 << sh) - 1)) | ((f >> sh) << (sh + a.tlog[m]));
}

// (xr, xi) fibres along mode m (padded extent P) times the 8x8-record
// complex matrix (re at Vr, im at Vr + 64; the tile's P x P block).  DIV:
// then divide every element by mu = sum_v lambda_v(i_v) (the last forward
// pass; returns true when a valid element has |mu| <= tiny)
template <int D, int P, bool DIV = false>
TSG_DEVINL bool fibre_cmode(const SolveArgs& a, const GD<D>& g, double* xr, double* xi, const double* Vr,
                            int ep, int m, const double* vh = nullptr) {
  const double* Vi = Vr + 64;
  const int shm = a.tsh[m];
  bool sing = false;
  for (int f = threadIdx.x; f < ep / P; f += THREADS) {
    const int lt0 = fibre_lt<D>(a, m, f);
    double zr[P], zi[P];
#pragma unroll
    for (int r = 0; r < P; ++r) {
      zr[r] = xr[lt0 + (r << shm)];
      zi[r] = xi[lt0 + (r << shm)];
    }
    // DIV: the eigenvalue sum of the fibre's other modes, once per fibre
    double br = 0.0, bi = 0.0;
    bool bvalid = true;
    if constexpr (DIV) {
#pragma unroll
      for (int v = 0; v < D; ++v) {
        if (v == m) continue;
        const int iv = (lt0 >> a.tsh[v]) & ((1 << a.tlog[v]) - 1);
        bvalid &= iv < g.ext[v];
        br += vh[v * VHS + 256 + iv];
        bi += vh[v * VHS + 264 + iv];
      }
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
      if constexpr (DIV) {
        const double mr = br + vh[m * VHS + 256 + r], mi = bi + vh[m * VHS + 264 + r];
        const double den = mr * mr + mi * mi;
        if (!(den > a.tiny * a.tiny)) {
          if (bvalid && r < g.ext[m]) sing = true;
          sr = si = 0.0;
        } else {
          const double inv = 1.0 / den, pr = sr, pi = si;
          sr = (pr * mr + pi * mi) * inv;
          si = (pi * mr - pr * mi) * inv;
        }
      }
      xr[lt0 + (r << shm)] = sr;
      xi[lt0 + (r << shm)] = si;
    }
  }
  return sing;
}

template <int D, int NB, int UB>
TSG_DEVINL void update_nb(const SolveArgs& a, const GD<D>& g, double* xr, const int64_t* goff, int ep, int m,
                          int klo, int khi) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int lpm = a.tlog[m], shm = a.tsh[m];
  const int cross = ep >> lpm;
  const int nblk = (cross + 7) >> 3;
  const int nm = a.dims[m];
  const int64_t sm = a.stride[m];
  const int row = g.start[m] + gq;  // B fragment: T_m[row][k], rows beyond the tile give 0
  const bool rok = gq < g.ext[m];
  // X(cross n, k) = X[goff[lt(n)] + (k - start_m) * stride_m]; padded cross
  // columns (goff < 0) are skipped
  const int64_t kofs = static_cast<int64_t>(klo + tq - g.start[m]) * sm;
  const int64_t s4 = 4 * sm;
  const double* pt0 = a.T[m] + row + static_cast<int64_t>(klo + tq) * nm;
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
      px[j] = a.X + (cok[j] ? go + kofs : 0);
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
    // C[g][2t+h]: cross column 8b + g, row 2t + h of mode m
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      if (!cok[j]) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 2 * tq + h;
        if (r < (1 << lpm)) xr[ltc[j] + (r << shm)] -= acc[j][h];
      }
    }
  }
}

#ifndef LAPD_NB
#define LAPD_NB 2
#endif
#ifndef LAPD_UBK
#define LAPD_UBK 4
#endif
// xr -= sum_k X(cross, k) T_m(rows, k) over rows k in [klo, khi) of mode m
// (cross-section of ep >> log2 P_m columns in 8-column blocks dealt to the
// warps, LAPD_NB blocks per round and LAPD_UBK k4-steps per load batch)
template <int D>
TSG_DEVINL void update_mode(const SolveArgs& a, const GD<D>& g, double* xr, const int64_t* goff, int ep, int m,
                            int klo, int khi) {
  update_nb<D, LAPD_NB, LAPD_UBK>(a, g, xr, goff, ep, m, klo, khi);
}

template <int D>
#ifndef LAPD_MINB
#define LAPD_MINB (2048 / EP + 1)  // 5 CTAs/SM at EP = 512 (96 registers)
#endif
__global__ void __launch_bounds__(THREADS, LAPD_MINB) solve_lapd_kernel(SolveArgs a) {
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) double xr[EP];
  __shared__ __align__(16) double xi[EP];
  __shared__ __align__(16) double vh[D * VHS];
  __shared__ int64_t goff[EP];  // global offset of each tile element (-1: padding)
  __shared__ GD<D> g;
  __shared__ int s_tile;
  const int tid = threadIdx.x;
  int ep = 1;
#pragma unroll
  for (int m = 0; m < D; ++m) ep <<= a.tlog[m];
  // optional cycle counters (TSG_PROF): 0 claim+geometry, 1 gather, 2 far
  // updates, 3 near updates (incl. flag waits), 4 base case, 5 scatter
  // (compiled in with -DLAPD_PROF=1 only: the counters cost registers)
#if LAPD_PROF
  unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tmark = clock64();
  auto mark = [&](int k) {
    if (a.prof) {
      const long long t = clock64();
      ph[k] += static_cast<unsigned long long>(t - tmark);
      tmark = t;
    }
  };
#else
  auto mark = [](int) {};
#endif
#if LAPD_PROF
  int ntl = 0;
#endif
  for (;;) {
#if LAPD_PROF
    ++ntl;
#endif
    mark(5);
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
      if (tid == 0) g.lt = a.order[qi];
    }
    __syncthreads();
    if (tid == 0) {
      int64_t gb = 0;
      for (int m = 0; m < D; ++m) gb += static_cast<int64_t>(g.start[m]) * a.stride[m];
      g.gbase = gb;
    }
    __syncthreads();

    mark(0);
    // ---- gather B~_t and the eigenvector bases ----
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
    }
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const double* src = a.vhat[m] + static_cast<int64_t>(g.tco[m]) * VHS;
      for (int e = 2 * tid; e < VHS; e += 2 * THREADS) cp_async16(vh + m * VHS + e, src + e, 16);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    mark(1);

    // ---- left-looking updates: far (tiles >= t+2), then near (t+1) ----
    int64_t mul = 1;
    int64_t muls[D];
#pragma unroll
    for (int m = 0; m < D; ++m) {
      muls[m] = mul;
      mul *= a.ntiles_mode[m];
    }
#ifndef LAPD_ONEPASS
#define LAPD_ONEPASS 1
#endif
    // LAPD_ONEPASS: wait for the t+1 flags and stream each mode's whole
    // range at once (half the update rounds; no overlap of the far rows with
    // the wait, which rarely matters on the wide hyperplanes of d = 6)
    constexpr int NPART = LAPD_ONEPASS ? 1 : 2;
    for (int part = 0; part < NPART && !(a.dbg & 4); ++part) {
      if (tid < D) {  // one thread per mode: the D flag round trips overlap
        const int m = tid;
        const int tm = g.tco[m], d0 = (part == 0 && !LAPD_ONEPASS) ? 2 : 1;
        if (tm + d0 < a.ntiles_mode[m]) waitp(a, g.lt + d0 * muls[m]);
      }
      __syncthreads();
#pragma unroll 1
      for (int m = 0; m < D; ++m) {
        const int tm = g.tco[m], p = a.ntiles_mode[m];
        int klo, khi;
        if (LAPD_ONEPASS) {
          klo = tm + 1 < p ? a.bnd[m][tm + 1] : 0;
          khi = tm + 1 < p ? a.dims[m] : 0;
        } else if (part == 0) {
          klo = tm + 2 < p ? a.bnd[m][tm + 2] : 0;
          khi = tm + 2 < p ? a.dims[m] : 0;
        } else {
          klo = tm + 1 < p ? a.bnd[m][tm + 1] : 0;
          khi = tm + 1 < p ? (tm + 2 < p ? a.bnd[m][tm + 2] : a.dims[m]) : 0;
        }
        if (khi > klo) update_mode<D>(a, g, xr, goff, ep, m, klo, khi);
        __syncthreads();
      }
      mark(2 + part);
    }

    // ---- diagonalised base case (complex, one thread per fibre) ----
    for (int pass = 0; pass < 2; ++pass) {  // 0: x V^-1 on every mode, 1: x V
#pragma unroll 1
      for (int m = 0; m < D; ++m) {
        const double* Vr = vh + m * VHS + (pass == 0 ? 0 : 128);
        if (pass == 0 && m == D - 1) {  // last forward pass: division by mu fused
          bool sing = false;
          switch (a.tlog[m]) {
            case 0: sing = fibre_cmode<D, 1, true>(a, g, xr, xi, Vr, ep, m, vh); break;
            case 1: sing = fibre_cmode<D, 2, true>(a, g, xr, xi, Vr, ep, m, vh); break;
            case 2: sing = fibre_cmode<D, 4, true>(a, g, xr, xi, Vr, ep, m, vh); break;
            default: sing = fibre_cmode<D, 8, true>(a, g, xr, xi, Vr, ep, m, vh); break;
          }
          if (sing) atomicMin(a.status, static_cast<int>(g.lt < 0x7f7f7f7e ? g.lt : 0x7f7f7f7e));
        } else {
          switch (a.tlog[m]) {
            case 0: fibre_cmode<D, 1>(a, g, xr, xi, Vr, ep, m); break;
            case 1: fibre_cmode<D, 2>(a, g, xr, xi, Vr, ep, m); break;
            case 2: fibre_cmode<D, 4>(a, g, xr, xi, Vr, ep, m); break;
            default: fibre_cmode<D, 8>(a, g, xr, xi, Vr, ep, m); break;
          }
        }
        __syncthreads();
      }
    }

    mark(4);
    // ---- scatter X_t (real part), release ----
    for (int l = tid; l < ep; l += THREADS) {
      const int64_t off = goff[l];
      if (off >= 0) a.X[off] = xr[l];
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(a.flags + g.lt, a.epoch);
    }
  }
#if LAPD_PROF
  if (a.prof && tid == 0) {
    for (int k = 0; k < 8; ++k) atomicAdd(a.prof + k, ph[k]);
    atomicAdd(a.prof + 8, static_cast<unsigned long long>(ntl));
  }
#endif
}

template <int D>
cudaError_t launch_d(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info) {
  auto k = solve_lapd_kernel<D>;
  int nsm = 0, occ = 0;
  if (cudaError_t e = kernel_setup(k, 0, THREADS, &nsm, &occ); e != cudaSuccess) return e;
  int64_t grid = static_cast<int64_t>(nsm) * occ;
  if (grid > a.ntiles) grid = a.ntiles;
  if (info) *info = SolveLaunchInfo{static_cast<int>(grid), THREADS, 0, occ};
  cudaError_t le = launch_pdl(k, static_cast<unsigned>(grid), THREADS, 0, st, a);
  return le != cudaSuccess ? le : cudaGetLastError();
}

}  // namespace

TileCaps solve_lapd_caps() { return TileCaps{8, EP, EP / 2}; }

cudaError_t launch_solve_lapd(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info) {
  if (a.ntiles <= 0) return cudaSuccess;
  switch (a.d) {
    case 4:
      return launch_d<4>(a, st, info);
    case 5:
      return launch_d<5>(a, st, info);
    case 6:
      return launch_d<6>(a, st, info);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace tsg
