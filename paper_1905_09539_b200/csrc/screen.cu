// Solvability screen on the GPU: the smallest
// |operator eigenvalue| over every eigenvalue tuple and its first position in
// the reference's odometer order (solvability.hpp:31-116, called at
// laplace.hpp:271-274 and gsylv.hpp:267-270 inside the reference's timed
// recursion).  O(prod n) scalar work: 191M tuples at C3, a few hundred
// microseconds here against seconds on the host cores.
//
//   Laplace:  lambda = ((lambda_0[i_0] + lambda_1[i_1]) + ...) + lambda_{d-1}[i_{d-1}],
//             tuple index L = i_0 + n_0 (i_1 + n_1 (...)), mode 0 fastest;
//   gsylv:    z = ((1 * mu_1[j_1]) * mu_2[j_2]) ...  over the tail modes, then
//             every diagonal block b of S: |S_bb + z T_bb| (1x1) or the
//             smaller eigenvalue magnitude of the 2x2 pencil block;
//             index L = b + n_blocks * (j_1 + n_1 (...)).
// The sums and products are formed in the reference's order (the inner
// partial sums / products once per inner index, then the last factor), so
// the values match the host screen to rounding of |.|; the first minimum
// (smallest L among equal values, the reference's strict `<` scan) comes
// from two passes: atomicMin of the value's bit pattern (non-negative
// doubles order like their bits), then atomicMin of L over the tuples
// attaining it.
#include <cstdint>
#include <cstring>

#include "common.cuh"
#include "screen.h"

namespace tsg {
namespace {

constexpr int kThreads = 256;

struct Cx {
  double re, im;
};
// rounded like the host's std::complex<double> arithmetic (no FMA contraction)
TSG_DEVINL Cx cadd(Cx a, Cx b) { return {__dadd_rn(a.re, b.re), __dadd_rn(a.im, b.im)}; }
TSG_DEVINL Cx cmul(Cx a, Cx b) {
  return {__dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, b.im)),
          __dadd_rn(__dmul_rn(a.re, b.im), __dmul_rn(a.im, b.re))};
}
TSG_DEVINL double cabs(Cx a) { return hypot(a.re, a.im); }
// principal square root
TSG_DEVINL Cx csqrt(Cx a) {
  const double r = cabs(a);
  double x = sqrt(0.5 * (r + fabs(a.re)));
  if (x == 0.0) return {0.0, 0.0};
  const double y = a.im / (2.0 * x);
  if (a.re >= 0.0) return {x, y};
  return {fabs(y), a.im >= 0.0 ? x : -x};
}

struct ScreenArgs {
  int d;              // lists folded into the "inner" array (Laplace: modes 0..d-2; gsylv: all tails)
  int n[8];           // extents of the eigenvalue lists
  const Cx* eig[8];   // eigenvalue lists (Laplace: all modes; gsylv: tails)
  int64_t ninner;     // prod of the inner extents
  Cx* inner;          // device: the partial sums (Laplace) / products (gsylv) in scan order
  int nouter;         // Laplace: n_{d-1} (the last mode's eigenvalues, eig[d]); gsylv: pencil blocks
  const Cx* outer;    // Laplace: the last mode's eigenvalues
  // gsylv pencil blocks
  const int* bstart;  // per block: first row
  const int* bsize;   // 1 or 2
  const double* S;    // n0 x n0 column-major
  const double* Tc;
  int n0;
  unsigned long long* key;  // [0] min value bits, [1] min index
};

// inner[p]: p decoded mode 0 fastest; Laplace ((0 + l_0) + l_1) + ..., gsylv ((1 * m_1) * m_2) ...
template <bool GS>
__global__ void inner_kernel(const ScreenArgs a) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < a.ninner;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    unsigned r = static_cast<unsigned>(p);
    Cx s = GS ? Cx{1.0, 0.0} : Cx{0.0, 0.0};
    for (int m = 0; m < a.d; ++m) {
      const unsigned q = r / static_cast<unsigned>(a.n[m]);
      const int i = static_cast<int>(r - q * static_cast<unsigned>(a.n[m]));
      r = q;
      s = GS ? cmul(s, a.eig[m][i]) : cadd(s, a.eig[m][i]);
    }
    a.inner[p] = s;
  }
}

// value of tuple (inner p, outer o): Laplace |inner[p] + lambda_{d-1}[o]|;
// gsylv: block o of the pencil S + z Tc with z = inner[p]
template <bool GS>
TSG_DEVINL double tuple_value(const ScreenArgs& a, Cx z, int o) {
  if (!GS) return cabs(cadd(z, a.outer[o]));
  const int i = a.bstart[o];
  const double* S = a.S;
  const double* T = a.Tc;
  const int n0 = a.n0;
  auto at = [&](const double* M, int r_, int c_) { return M[r_ + static_cast<int64_t>(c_) * n0]; };
  // C(s) + z * t, t real: (s + z.re t, z.im t)
  auto pen = [&](int r_, int c_) {
    const double t = at(T, r_, c_);
    return Cx{__dadd_rn(at(S, r_, c_), __dmul_rn(z.re, t)), __dmul_rn(z.im, t)};
  };
  if (a.bsize[o] == 1) return cabs(pen(i, i));
  const Cx m00 = pen(i, i), m01 = pen(i, i + 1), m11 = pen(i + 1, i + 1);
  const Cx m10{at(S, i + 1, i), 0.0};
  const Cx sm = cadd(m00, m11);
  const Cx h{__dmul_rn(0.5, sm.re), __dmul_rn(0.5, sm.im)};
  const Cx p1 = cmul(m00, m11), p2 = cmul(m01, m10);
  const Cx det{__dsub_rn(p1.re, p2.re), __dsub_rn(p1.im, p2.im)};
  const Cx hh = cmul(h, h);
  const Cx rt = csqrt(Cx{__dsub_rn(hh.re, det.re), __dsub_rn(hh.im, det.im)});
  return fmin(cabs(cadd(h, rt)), cabs(Cx{__dsub_rn(h.re, rt.re), __dsub_rn(h.im, rt.im)}));
}

// Scan order: Laplace L = p + ninner * o (the last mode slowest); gsylv
// L = o + nblk * p (blocks fastest).  Each thread owns inner indices p.
template <bool GS>
TSG_DEVINL int64_t lin(const ScreenArgs& a, int64_t p, int o) {
  return GS ? static_cast<int64_t>(o) + static_cast<int64_t>(a.nouter) * p : p + a.ninner * o;
}

template <bool GS>
__global__ void __launch_bounds__(kThreads) min_kernel(const ScreenArgs a) {
  double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  for (int64_t p = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; p < a.ninner;
       p += static_cast<int64_t>(gridDim.x) * kThreads) {
    const Cx z = a.inner[p];
    for (int o = 0; o < a.nouter; ++o) best = fmin(best, tuple_value<GS>(a, z, o));
  }
  for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
  __shared__ double wb[kThreads / 32];
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kThreads / 32; ++w) best = fmin(best, wb[w]);
    atomicMin(a.key, static_cast<unsigned long long>(__double_as_longlong(best)));
  }
}

template <bool GS>
__global__ void __launch_bounds__(kThreads) argmin_kernel(const ScreenArgs a) {
  const unsigned long long vkey = *a.key;
  unsigned long long first = ~0ull;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; p < a.ninner;
       p += static_cast<int64_t>(gridDim.x) * kThreads) {
    const Cx z = a.inner[p];
    for (int o = 0; o < a.nouter; ++o)
      if (static_cast<unsigned long long>(__double_as_longlong(tuple_value<GS>(a, z, o))) == vkey) {
        const unsigned long long L = static_cast<unsigned long long>(lin<GS>(a, p, o));
        first = L < first ? L : first;
        break;  // the smallest o of this p gives its smallest L in both orders
      }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, first, o);
    first = v < first ? v : first;
  }
  if ((threadIdx.x & 31) == 0 && first != ~0ull) atomicMin(a.key + 1, first);
}

template <bool GS>
cudaError_t run(ScreenArgs& a, int nsm, cudaStream_t st) {
  const int64_t want = (a.ninner + kThreads - 1) / kThreads;
  const int grid = static_cast<int>(want < 16LL * nsm ? (want > 0 ? want : 1) : 16LL * nsm);
  inner_kernel<GS><<<grid, kThreads, 0, st>>>(a);
  min_kernel<GS><<<grid, kThreads, 0, st>>>(a);
  argmin_kernel<GS><<<grid, kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t screen_min(const ScreenSpec& sp, cudaStream_t st, double* min_abs, int64_t* index) {
  ScreenArgs a{};
  const bool gs = sp.S != nullptr;
  // Laplace: inner = modes 0..d-2, outer = the last mode; gsylv: inner = every tail, outer = the blocks
  a.d = gs ? sp.nlists : sp.nlists - 1;
  a.ninner = 1;
  size_t neig = 0;
  for (int m = 0; m < sp.nlists; ++m) {
    a.n[m] = sp.n[m];
    neig += sp.n[m];
    if (m < a.d) a.ninner *= sp.n[m];
  }
  if (a.ninner >= (int64_t{1} << 31)) return cudaErrorInvalidValue;
  a.nouter = gs ? sp.nblk : sp.n[sp.nlists - 1];
  if (gs) a.n0 = sp.n0;
  const size_t bytes_eig = neig * sizeof(Cx);
  const size_t nn = gs ? static_cast<size_t>(sp.n0) * sp.n0 : 0;
  const size_t bytes = 2 * sizeof(unsigned long long) + bytes_eig + static_cast<size_t>(a.ninner) * sizeof(Cx) +
                       2 * nn * sizeof(double) + (gs ? 2 * sp.nblk * sizeof(int) : 0);
  char* buf = nullptr;
  cudaError_t e = cudaMallocAsync(&buf, bytes, st);
  if (e != cudaSuccess) return e;
  char* p = buf;
  a.key = reinterpret_cast<unsigned long long*>(p);
  p += 2 * sizeof(unsigned long long);
  const unsigned long long init[2] = {~0ull, ~0ull};
  e = cudaMemcpyAsync(a.key, init, sizeof(init), cudaMemcpyHostToDevice, st);
  size_t off = 0;
  for (int m = 0; m < sp.nlists && e == cudaSuccess; ++m) {
    a.eig[m] = reinterpret_cast<const Cx*>(p) + off;
    e = cudaMemcpyAsync(reinterpret_cast<Cx*>(p) + off, sp.eig_re_im[m], sp.n[m] * sizeof(Cx),
                        cudaMemcpyHostToDevice, st);
    off += sp.n[m];
  }
  if (!gs) a.outer = a.eig[sp.nlists - 1];
  p += bytes_eig;
  a.inner = reinterpret_cast<Cx*>(p);
  p += static_cast<size_t>(a.ninner) * sizeof(Cx);
  if (gs && e == cudaSuccess) {
    double* dS = reinterpret_cast<double*>(p);
    double* dT = dS + nn;
    int* bs = reinterpret_cast<int*>(dT + nn);
    int* bz = bs + sp.nblk;
    e = cudaMemcpyAsync(dS, sp.S, nn * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dT, sp.Tc, nn * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(bs, sp.bstart, sp.nblk * sizeof(int), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(bz, sp.bsize, sp.nblk * sizeof(int), cudaMemcpyHostToDevice, st);
    a.S = dS;
    a.Tc = dT;
    a.bstart = bs;
    a.bsize = bz;
  }
  if (e == cudaSuccess) e = gs ? run<true>(a, sp.nsm, st) : run<false>(a, sp.nsm, st);
  unsigned long long h[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, a.key, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaError_t e2 = cudaFreeAsync(buf, st);
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  std::memcpy(min_abs, &h[0], sizeof(double));
  *index = static_cast<int64_t>(h[1]);
  return cudaSuccess;
}

}  // namespace tsg
