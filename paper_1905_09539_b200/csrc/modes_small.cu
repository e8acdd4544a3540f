// Fused transforms of small modes (n <= 48): Y = X x_a A x_b B for two
// consecutive modes a, b = a + 1 (or one mode, B = null) in ONE pass over
// HBM.  For C3 (24^6) the per-mode DGEMM is HBM-bound at n/8 = 3 FLOP/B with
// badly padded 64-wide tiles; pairing the modes halves the passes and the
// per-fibre products run from shared memory.
//
// Block = (c inner indices) x (n_a x n_b group) x (o outer indices), staged
// in shared memory in that order (inner fastest): c consecutive indices of
// the contiguous prefix (modes < a) when a > 0, else o consecutive indices
// of the suffix (modes > b), so every block is a few contiguous runs.  Each
// warp owns whole 8-fibre groups along the mode being applied (in place:
// DMMA accumulators, written back once the group's rows are read), with the
// n x n matrices as register fragments.  Rows of c * n_a doubles are padded
// to 4 (mod 8) doubles in shared memory, so the four k of a DMMA step of
// mode b (c * n_a apart, a multiple of 8 doubles) fall on distinct banks;
// results go back as 16-byte stores of two neighbouring fibres.
// Reference: mode_multiply (tensor.hpp:187-231) at laplace.hpp:282/297.
#include <cstdint>
#include <cstdio>

#include "common.cuh"
#include "gemm.h"
#include "util.h"

namespace tsg {
namespace {

constexpr int THREADS = 256;
#ifndef PAIR_PROF
#define PAIR_PROF 0
#endif
#if PAIR_PROF
// development: per-phase cycle counters of pair_kernel (tools/mkalt.py <name> -DPAIR_PROF=1)
__device__ unsigned long long g_pair_prof[8];
#define PP_T(v) const long long v = clock64()
#define PP_ADD(k, t0) (pph[k] += clock64() - (t0))
#else
#define PP_T(v)
#define PP_ADD(k, t0)
#endif

struct PairArgs {
  const double* X;
  double* Y;
  const double* A;  // n_a x n_a, column-major (Y = X x_a A: y_i = sum_k A(i,k) x_k)
  const double* B;  // n_b x n_b or null
  int na, nb;       // nb = 1 when B is null
  int c, o;         // block inner / outer extents (c a power of two)
  int lc;           // log2 c
  int64_t P, Q;     // prefix (modes < a) and suffix (modes > b) sizes
  int64_t nblk;     // blocks
  int bsz;          // doubles per block = c * na * nb * o
  int row, pitch;   // c * na and its padded pitch in shared memory (4 mod 8 doubles)
  int vec;          // 16-byte chunks (runs of even length at even offsets)
};

// y[f, i] = sum_k M(i, k) x[f, k] for the fibres of the block along one
// coordinate: fibre f = lo + lext * hi sits at blk + lo + hstr * hi and its
// element k at + kstr * k.  DMMA: M (N x N, registers) is the A operand,
// each warp takes whole 8-fibre groups (B operand from shared memory) and
// writes them back in place once all their rows are read.
// POW2: lext = 1 << llog (mode a: the prefix chunk c), any value; otherwise
// lext is a multiple of 8 (mode b: c * n_a), a group never straddles two hi
// and (lo, hi) advance incrementally — no integer division in the loop.
// When lext is even, fibres 2t and 2t + 1 of a group are neighbours in
// memory and a lane stores its two accumulator columns as one 16-byte word.
template <int N, bool POW2>
TSG_DEVINL void fibres(double* blk, const double* M, int lext, int llog, int kstr, int hstr, int nf) {
  constexpr int RB = N / 8, KS = N / 4;
  // N <= 32: the matrix fragments live in registers; larger N reads them
  // from shared memory per k-step (conflict-free: N = 8 mod 32 for 40)
  constexpr bool REG = N <= 32;
  constexpr int KR = REG ? KS : 1;
  constexpr int NW = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  double af[RB][KR];
  if constexpr (REG) {
#pragma unroll
    for (int rb = 0; rb < RB; ++rb)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) af[rb][ks] = M[(8 * rb + gq) + N * (4 * ks + tq)];
  }
  const bool pairst = POW2 ? (lext >= 2) : true;
  // group base (fibre 8 fb) of this warp, advanced by NW groups per round
  int lo = 0, hi = 0;
  if constexpr (!POW2) {
    lo = 8 * warp;
    while (lo >= lext) lo -= lext, ++hi;
  }
  for (int fb = warp; fb < (nf >> 3); fb += NW) {
    // fibre of this lane as B column: f = 8 fb + gq; as C columns: 8 fb + 2 tq (+ 1)
    int oB, oC0, oC1;
    if constexpr (POW2) {
      const int fB = 8 * fb + gq, fC = 8 * fb + 2 * tq;
      oB = (fB & (lext - 1)) + hstr * (fB >> llog);
      oC0 = (fC & (lext - 1)) + hstr * (fC >> llog);
      oC1 = ((fC + 1) & (lext - 1)) + hstr * ((fC + 1) >> llog);
    } else {
      const int g0 = lo + hstr * hi;
      oB = g0 + gq;
      oC0 = g0 + 2 * tq;
      oC1 = oC0 + 1;
      lo += 8 * NW;
      while (lo >= lext) lo -= lext, ++hi;
    }
    const double* pB = blk + oB + kstr * tq;
    double bf[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bf[ks] = pB[kstr * 4 * ks];
    double c[RB][2];
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) c[rb][0] = c[rb][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        if constexpr (REG) dmma(c[rb][0], c[rb][1], af[rb][ks], bf[ks]);
        else dmma(c[rb][0], c[rb][1], M[(8 * rb + gq) + N * (4 * ks + tq)], bf[ks]);
      }
    __syncwarp();  // every row of the warp's 8 fibres has been read
    if (pairst) {
      double* pC = blk + oC0 + kstr * gq;
#pragma unroll
      for (int rb = 0; rb < RB; ++rb)
        *reinterpret_cast<double2*>(pC + kstr * 8 * rb) = make_double2(c[rb][0], c[rb][1]);
    } else {
      double* pC0 = blk + oC0 + kstr * gq;
      double* pC1 = blk + oC1 + kstr * gq;
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        pC0[kstr * 8 * rb] = c[rb][0];
        pC1[kstr * 8 * rb] = c[rb][1];
      }
    }
    __syncwarp();
  }
}

// Double-buffered: while the fibres of block b are multiplied in shared
// memory, block b + grid streams into the other buffer (cp.async, 16-byte
// chunks when the block's contiguous runs allow), so HBM traffic overlaps
// the DMMA work; results go back with 16-byte stores.
template <int NA, int NB>
__global__ void __launch_bounds__(THREADS) pair_kernel(PairArgs g) {
  extern __shared__ __align__(16) double sm[];
  double* ma = sm;
  double* mb = sm + NA * NA;
  double* buf0 = mb + (NB > 1 ? NB * NB : 0);
  for (int e = threadIdx.x; e < NA * NA; e += THREADS) ma[e] = g.A[e];
  if (NB > 1)
    for (int e = threadIdx.x; e < NB * NB; e += THREADS) mb[e] = g.B[e];
  const int c = g.c, o = g.o;
  constexpr int GRP = NA * NB;
  const int64_t npc = g.P / c;
  // Block element e (dense order ic, ia, ib, io) = x + row * r with
  // x = ic + c * ia < row = c * NA and r = ib + NB * io: it lives at
  // x + pitch * r in shared memory and at base + ic + P * (ia + NA * r) in
  // the tensor.  Runs of c consecutive elements are contiguous, as is the
  // whole block when P == 1, so pairs (e, e + 1) with e even are 16-byte
  // chunks.  A thread's elements are `step` apart and c divides step, so
  // ic is fixed per thread and the tensor offset is an arithmetic
  // progression (a wrap of x moves ia by -NA and r by +1: no change); the
  // shared offset gains the row padding on a wrap.  No division per element.
  const int row = g.row, pitch = g.pitch, pad = pitch - row;
  const int bufsz = pitch * (g.bsz / row);
  const bool vec = g.vec != 0;
  const int step = vec ? 2 * THREADS : THREADS;
  const int dx = step % row, dr = step / row;
  const int e0 = vec ? 2 * threadIdx.x : threadIdx.x;
  const int x0 = e0 % row, r0 = e0 / row;
  const int s0 = x0 + pitch * r0, ds = dx + pitch * dr;
  const int64_t g0 = (x0 & (c - 1)) + g.P * ((x0 >> g.lc) + static_cast<int64_t>(NA) * r0);
  const int64_t dg = g.P * ((dx >> g.lc) + static_cast<int64_t>(NA) * dr);
  auto base_of = [&](int64_t bk) {
    const int64_t pc = bk % npc, sc = bk / npc;
    return pc * c + sc * static_cast<int64_t>(o) * g.P * GRP;
  };
  auto gather = [&](int64_t bk, double* blk) {
    const double* src = g.X + base_of(bk) + g0;
    double* dstp = blk + s0;
    int x = x0;
    for (int e = e0; e < g.bsz; e += step) {
      if (vec) cp_async16(dstp, src, 16);
      else cp_async8(dstp, src, 8);
      src += dg, dstp += ds, x += dx;
      if (x >= row) x -= row, dstp += pad;
    }
    cp_async_commit();
  };
  int64_t bk = blockIdx.x;
#if PAIR_PROF
  long long pph[8] = {};
#endif
  if (bk < g.nblk) gather(bk, buf0);
  for (int it = 0; bk < g.nblk; bk += gridDim.x, ++it) {
    double* blk = buf0 + (it & 1) * bufsz;
    double* nxt = buf0 + ((it + 1) & 1) * bufsz;
    const int64_t bn = bk + gridDim.x;
    PP_T(t0);
    if (bn < g.nblk) gather(bn, nxt);  // the other buffer was scattered last round
    else cp_async_commit();
    PP_ADD(0, t0);
    PP_T(t1);
    cp_async_wait<1>();
    PP_ADD(1, t1);
    PP_T(t2);
    __syncthreads();
    PP_ADD(2, t2);
    PP_T(t3);
    // mode a: fibres (ic; ib, io), rows c apart
    fibres<NA, true>(blk, ma, c, g.lc, c, pitch, g.bsz / NA);
    PP_ADD(3, t3);
    if constexpr (NB > 1) {
      PP_T(t4);
      __syncthreads();
      PP_ADD(2, t4);
      PP_T(t5);
      // mode b: fibres (ic, ia; io), rows one pitch apart (row = c * NA, a multiple of 8)
      fibres<NB, false>(blk, mb, row, 0, pitch, pitch * NB, g.bsz / NB);
      PP_ADD(4, t5);
    }
    PP_T(t6);
    __syncthreads();
    PP_ADD(2, t6);
    PP_T(t7);
    double* dst = g.Y + base_of(bk) + g0;
    const double* srcp = blk + s0;
    int x = x0;
    for (int e = e0; e < g.bsz; e += step) {
      if (vec) *reinterpret_cast<double2*>(dst) = *reinterpret_cast<const double2*>(srcp);
      else *dst = *srcp;
      dst += dg, srcp += ds, x += dx;
      if (x >= row) x -= row, srcp += pad;
    }
    PP_ADD(5, t7);
    PP_T(t8);
    __syncthreads();  // blk is the next round's prefetch target
    PP_ADD(2, t8);
#if PAIR_PROF
    pph[6] += 1;
#endif
  }
  cp_async_wait_all();
#if PAIR_PROF
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < 7; ++k) atomicAdd(&g_pair_prof[k], static_cast<unsigned long long>(pph[k]));
#endif
}

template <int NA, int NB>
cudaError_t launch_pair(const PairArgs& g, cudaStream_t st) {
  const int smem = (NA * NA + (NB > 1 ? NB * NB : 0) + 2 * g.pitch * (g.bsz / g.row)) * 8;
  auto k = pair_kernel<NA, NB>;
  int nsm = 0, occ = 0;
  if (cudaError_t e = kernel_setup(k, smem, THREADS, &nsm, &occ); e != cudaSuccess) return e;
  int64_t grid = static_cast<int64_t>(nsm) * occ;
  if (grid > g.nblk) grid = g.nblk;
#if PAIR_PROF
  unsigned long long z[8] = {};
  cudaMemcpyToSymbolAsync(g_pair_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
#endif
  k<<<static_cast<unsigned>(grid), THREADS, smem, st>>>(g);
#if PAIR_PROF
  unsigned long long h[8];
  cudaMemcpyFromSymbolAsync(h, g_pair_prof, sizeof(h), 0, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  const double nb = h[6] ? static_cast<double>(h[6]) : 1.0;
  std::fprintf(stderr, "[tsg profp] %dx%d c=%d o=%d vec=%d grid=%lld smem=%d | per block per warp (cycles): gather issue %.0f  "
               "cp.async wait %.0f  barriers %.0f  mode a %.0f  mode b %.0f  scatter %.0f  (blocks x warps %.0f)\n",
               NA, NB, g.c, g.o, g.vec, static_cast<long long>(grid), smem, h[0] / nb, h[1] / nb, h[2] / nb, h[3] / nb,
               h[4] / nb, h[5] / nb, nb);
#endif
  return cudaGetLastError();
}

template <int NA>
cudaError_t dispatch_b(const PairArgs& g, cudaStream_t st) {
  switch (g.nb) {
    case 1: return launch_pair<NA, 1>(g, st);
    case 16: return launch_pair<NA, 16>(g, st);
    case 24: return launch_pair<NA, 24>(g, st);
    case 32: return launch_pair<NA, 32>(g, st);
    case 40: return launch_pair<NA, 40>(g, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

bool small_mode_ok(int n) { return n == 16 || n == 24 || n == 32 || n == 40; }

namespace {
// measured best of 3K / 4.6K / 6.9K doubles per block buffer
constexpr int kBlockTarget = 6912;
static_assert((40 * 40 * 2 + 2 * (kBlockTarget + 4 * (kBlockTarget / 16))) * 8 <= 227 * 1024,
              "largest fused pass must fit the sm_100a shared-memory opt-in");
// Block shape of a fused pass: c | P (inner chunk of the prefix), o | Q
// (outer batch), powers of two, at most kBlockTarget doubles per block
// (two buffers: up to (40^2 + 40^2 + 2 * 6912) * 8 B = 136 KB of shared
// memory for the 40x40 pair, one CTA per SM; 16x16 pairs ~110 KB).  The fibre
// products work on whole 8-fibre blocks, so the fibres per block along
// mode a (c * nb * o) and mode b (c * na * o) must be multiples of 8: pairs
// always are (extents 16..40); a single mode may need o > 1 (odd prefix) and
// is unsupported when neither P nor Q supplies the factor (GEMM then).
bool pass_shape(int64_t P, int64_t Q, int na, int nb, int* c_out, int* o_out) {
  const int grp = na * nb;
  const int target = kBlockTarget;
  int c = 1, o = 1;
  if (P > 1) {
    while (c * 2 * grp <= target && P % (c * 2) == 0 && c * 2 <= THREADS) c *= 2;  // c | THREADS: see pair_kernel
  } else {
    while (o * 2 * grp <= target && Q % (o * 2) == 0) o *= 2;
  }
  auto ok = [&] { return (c * nb * o) % 8 == 0 && (nb == 1 || (c * na * o) % 8 == 0); };
  while (!ok() && Q % (o * 2) == 0 && c * grp * o * 2 <= target) o *= 2;  // stay within the block budget
  if (!ok()) return false;
  *c_out = c;
  *o_out = o;
  return true;
}
}  // namespace

bool small_pass_ok(int d, const int* dims, int a, bool pair) {
  const int b = pair ? a + 1 : a;
  if (a < 0 || b >= d || !small_mode_ok(dims[a]) || (pair && !small_mode_ok(dims[b]))) return false;
  int64_t P = 1, Q = 1;
  for (int v = 0; v < a; ++v) P *= dims[v];
  for (int v = b + 1; v < d; ++v) Q *= dims[v];
  int c, o;
  return pass_shape(P, Q, dims[a], pair ? dims[b] : 1, &c, &o);
}

cudaError_t mode_pair_small(const double* X, double* Y, int d, const int* dims, int a, bool pair,
                            const double* A, const double* B, cudaStream_t st, double* flops) {
  const int b = pair ? a + 1 : a;
  if (a < 0 || b >= d || !small_mode_ok(dims[a]) || (pair && !small_mode_ok(dims[b])))
    return cudaErrorInvalidValue;
  PairArgs g{};
  g.X = X;
  g.Y = Y;
  g.A = A;
  g.B = pair ? B : nullptr;
  g.na = dims[a];
  g.nb = pair ? dims[b] : 1;
  g.P = 1;
  g.Q = 1;
  for (int v = 0; v < a; ++v) g.P *= dims[v];
  for (int v = b + 1; v < d; ++v) g.Q *= dims[v];
  const int grp = g.na * g.nb;
  if (!pass_shape(g.P, g.Q, g.na, g.nb, &g.c, &g.o)) return cudaErrorNotSupported;
  g.bsz = g.c * grp * g.o;
  g.row = g.c * g.na;
  g.pitch = g.row + (4 - g.row % 8 + 8) % 8;   // 4 (mod 8) doubles: see the header
  g.lc = 0;
  while ((1 << g.lc) < g.c) ++g.lc;
  g.nblk = (g.P / g.c) * (g.Q / g.o);
  g.vec = ((g.c % 2 == 0 && g.P % 2 == 0) || (g.c == 1 && g.P == 1 && grp % 2 == 0)) &&
          (reinterpret_cast<uintptr_t>(X) & 15) == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  if (flops) *flops += 2.0 * static_cast<double>(g.P) * g.Q * grp * (g.na + g.nb - (pair ? 0 : 1));
  switch (g.na) {
    case 16: return dispatch_b<16>(g, st);
    case 24: return dispatch_b<24>(g, st);
    case 32: return dispatch_b<32>(g, st);
    case 40: return dispatch_b<40>(g, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tsg
