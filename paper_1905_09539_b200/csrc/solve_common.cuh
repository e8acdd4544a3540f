// Shared pieces of the dataflow solve kernels (solve.cu, solve_lap.cu):
// complex helpers and the DMMA left-looking update pass.
#pragma once
#include <cstdint>

#include "common.cuh"
#include "solve.h"

namespace tsg {
namespace {

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
// Left-looking update pass over one contiguous K range of mode m:
//   dst -= sign * sum_j coef_j[rows of t along m, k_lo:k_hi] x_m src_j[k_lo:k_hi]
// (sign = -1 subtracts; gsylv W partials accumulate with +1).  The K range
// is either the "far" tiles t_m+2.. (ready long before) or the nearest tile
// t_m+1, so one flag wait covers the whole pass.  The accumulator (dst
// restricted to the tile: M = e_m rows x N = E/e_m cross-section columns)
// lives in registers across an NSTAGE-deep cp.async ring of K chunks.
// ---------------------------------------------------------------------------
template <int D, typename C, typename TG>
__device__ __noinline__ void update_pass(const SolveArgs& a, const TG& tg, double* smem, double* dst,
                            int m, int k_lo, int k_hi, int64_t wait_tile,
                            const double* coef0, const double* src0,
                            const double* coef1, const double* src1, int nsrc, double sign) {
  if (k_hi <= k_lo) return;  // uniform
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int em = tg.ext[m];
  const int P = tg.tstride[m];
  const int N = tg.E / em;
  const int NB = (N + 7) >> 3;
  const int NP = NB * 8;
  const int MBv = (em + 7) >> 3;
  const int nm = a.dims[m];
  const int64_t sm_stride = a.stride[m];
  int64_t* csoff = reinterpret_cast<int64_t*>(smem + C::OFF_CS);
  double* sB = smem + C::OFF_B;
  double* sA = smem + C::OFF_A;

  if (tid == 0 && wait_tile >= 0) {
    const int* f = a.flags + wait_tile;
    while (ld_acquire(f) < a.epoch) __nanosleep(32);
  }
  // Cross-section offsets (modes != m, mode 0 fastest) of the tile.
  for (int n = tid; n < N; n += C::THREADS) {
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

  double c[C::MB][C::NBW][2];
#pragma unroll
  for (int ib = 0; ib < C::MB; ++ib)
#pragma unroll
    for (int jj = 0; jj < C::NBW; ++jj)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = ib * 8 + gq, n = (warp + (C::THREADS / 32) * jj) * 8 + 2 * tq + h;
        double v = 0.0;
        if (ib < MBv && i < em && n < N) {
          const int q = n / P, p = n - q * P;
          v = dst[p + i * P + q * P * em];
        }
        c[ib][jj][h] = v;
      }

  const int kr = k_hi - k_lo;
  const int nck = (kr + C::KC - 1) / C::KC;  // chunks per source
  const int nchunks = nck * nsrc;
  const int row0 = tg.start[m];
  auto issue = [&](int ci, int buf) {
    const int j = ci / nck;
    const int k0 = k_lo + (ci - j * nck) * C::KC;
    const int kv = min(C::KC, k_hi - k0);
    const double* coef = j == 0 ? coef0 : coef1;
    const double* src = j == 0 ? src0 : src1;
    double* A = sA + buf * C::STAGE_A;
    double* B = sB + buf * C::STAGE_B;
    for (int e = tid; e < C::KC * C::MPAD; e += C::THREADS) {
      const int k = e / C::MPAD, i = e - k * C::MPAD;
      const bool ok = (i < em) && (k < kv);
      cp_async8(A + k * C::LDA + i,
                ok ? coef + (row0 + i) + static_cast<int64_t>(k0 + k) * nm : coef, ok ? 8 : 0);
    }
    if (m == 0) {
      for (int e = tid; e < C::KC * NP; e += C::THREADS) {
        const int n = e / C::KC, k = e - n * C::KC;
        const bool ok = (k < kv) && (n < N);
        cp_async8(B + k * C::LDB + n,
                  ok ? src + csoff[n] + static_cast<int64_t>(k0 + k) * sm_stride : src, ok ? 8 : 0);
      }
    } else {
      for (int e = tid; e < C::KC * NP; e += C::THREADS) {
        const int k = e / NP, n = e - k * NP;
        const bool ok = (k < kv) && (n < N);
        cp_async8(B + k * C::LDB + n,
                  ok ? src + csoff[n] + static_cast<int64_t>(k0 + k) * sm_stride : src, ok ? 8 : 0);
      }
    }
  };

#pragma unroll
  for (int st = 0; st < C::NSTAGE - 1; ++st) {
    if (st < nchunks) issue(st, st);
    cp_async_commit();
  }
  for (int ci = 0; ci < nchunks; ++ci) {
    cp_async_wait<C::NSTAGE - 2>();
    __syncthreads();
    {
      const int nx = ci + C::NSTAGE - 1;
      if (nx < nchunks) issue(nx, nx % C::NSTAGE);
      cp_async_commit();
    }
    const int buf = ci % C::NSTAGE;
    const double* A = sA + buf * C::STAGE_A;
    const double* B = sB + buf * C::STAGE_B;
#pragma unroll
    for (int k4 = 0; k4 < C::KC; k4 += 4) {
      double af[C::MB], bf[C::NBW];
#pragma unroll
      for (int ib = 0; ib < C::MB; ++ib) af[ib] = sign * A[(k4 + tq) * C::LDA + ib * 8 + gq];
#pragma unroll
      for (int jj = 0; jj < C::NBW; ++jj) {
        const int jb = warp + (C::THREADS / 32) * jj;
        bf[jj] = (jb < NB) ? B[(k4 + tq) * C::LDB + jb * 8 + gq] : 0.0;
      }
#pragma unroll
      for (int ib = 0; ib < C::MB; ++ib) {
        if (ib >= MBv) continue;
#pragma unroll
        for (int jj = 0; jj < C::NBW; ++jj) {
          if (warp + (C::THREADS / 32) * jj >= NB) continue;
          dmma(c[ib][jj][0], c[ib][jj][1], af[ib], bf[jj]);
        }
      }
    }
  }
  cp_async_wait_all();

#pragma unroll
  for (int ib = 0; ib < C::MB; ++ib)
#pragma unroll
    for (int jj = 0; jj < C::NBW; ++jj)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = ib * 8 + gq, n = (warp + (C::THREADS / 32) * jj) * 8 + 2 * tq + h;
        if (ib < MBv && i < em && n < N) {
          const int q = n / P, p = n - q * P;
          dst[p + i * P + q * P * em] = c[ib][jj][h];
        }
      }
  __syncthreads();
}


}  // namespace
}  // namespace tsg
