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
// thread owns whole fibres along the mode being applied (in place, the
// fibre lives in registers), with the n x n matrices in shared memory.
// Reference: mode_multiply (tensor.hpp:187-231) at laplace.hpp:282/297.
#include <cstdint>

#include "common.cuh"
#include "gemm.h"
#include "util.h"

namespace tsg {
namespace {

constexpr int THREADS = 256;

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
  int vec;          // 16-byte chunks (runs of even length at even offsets)
};

// y[f, i] = sum_k M(i, k) x[f, k] for the fibres of the block along a
// coordinate of extent N and stride st (in the block): fibre index f
// enumerates (lo < st) x (hi) with element offset lo + st * (k + N * hi).
// DMMA: M (N x N, registers) is the A operand, each warp takes whole
// 8-fibre blocks (B operand from shared memory) and writes them back in
// place once all their rows are read.
template <int N>
TSG_DEVINL void fibres(double* blk, const double* M, int st, int nf) {
  constexpr int RB = N / 8, KS = N / 4;
  // N <= 32: the matrix fragments live in registers; larger N reads them
  // from shared memory per k-step (conflict-free: N = 8 mod 32 for 40)
  constexpr bool REG = N <= 32;
  constexpr int KR = REG ? KS : 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  double af[RB][KR];
  if constexpr (REG) {
#pragma unroll
    for (int rb = 0; rb < RB; ++rb)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) af[rb][ks] = M[(8 * rb + gq) + N * (4 * ks + tq)];
  }
  for (int fb = warp; fb < (nf >> 3); fb += THREADS / 32) {
    // fibre of this lane as B column: f = 8 fb + gq; as C column: 8 fb + 2 tq + h
    const int fB = 8 * fb + gq;
    const double* pB = blk + (fB % st) + static_cast<int64_t>(st) * N * (fB / st);
    double bf[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bf[ks] = pB[st * (4 * ks + tq)];
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
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int fC = 8 * fb + 2 * tq + h;
      double* pC = blk + (fC % st) + static_cast<int64_t>(st) * N * (fC / st);
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) pC[st * (8 * rb + gq)] = c[rb][h];
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
  // element e of a block: (ic, gi, io) at base + ic + P * (gi + GRP * io);
  // runs of c consecutive elements are contiguous, as is the whole block
  // when P == 1, so pairs (e, e + 1) with e even are 16-byte chunks
  const bool vec = g.vec != 0;
  auto base_of = [&](int64_t bk) {
    const int64_t pc = bk % npc, sc = bk / npc;
    return pc * c + sc * static_cast<int64_t>(o) * g.P * GRP;
  };
  auto off_of = [&](int e) {
    const int ic = e & (c - 1), rest = e >> g.lc;
    const int gi = rest % GRP, io = rest / GRP;
    return ic + g.P * (gi + static_cast<int64_t>(GRP) * io);
  };
  auto gather = [&](int64_t bk, double* blk) {
    const int64_t base = base_of(bk);
    if (vec) {
      for (int e = 2 * threadIdx.x; e < g.bsz; e += 2 * THREADS) cp_async16(blk + e, g.X + base + off_of(e), 16);
    } else {
      for (int e = threadIdx.x; e < g.bsz; e += THREADS) cp_async8(blk + e, g.X + base + off_of(e), 8);
    }
    cp_async_commit();
  };
  int64_t bk = blockIdx.x;
  if (bk < g.nblk) gather(bk, buf0);
  for (int it = 0; bk < g.nblk; bk += gridDim.x, ++it) {
    double* blk = buf0 + (it & 1) * g.bsz;
    double* nxt = buf0 + ((it + 1) & 1) * g.bsz;
    const int64_t bn = bk + gridDim.x;
    if (bn < g.nblk) gather(bn, nxt);  // the other buffer was scattered last round
    else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    fibres<NA>(blk, ma, c, g.bsz / NA);  // mode a: stride c in the block
    if constexpr (NB > 1) {
      __syncthreads();
      fibres<NB>(blk, mb, c * NA, g.bsz / NB);
    }
    __syncthreads();
    const int64_t base = base_of(bk);
    if (vec) {
      for (int e = 2 * threadIdx.x; e < g.bsz; e += 2 * THREADS)
        *reinterpret_cast<double2*>(g.Y + base + off_of(e)) = *reinterpret_cast<const double2*>(blk + e);
    } else {
      for (int e = threadIdx.x; e < g.bsz; e += THREADS) g.Y[base + off_of(e)] = blk[e];
    }
    __syncthreads();  // blk is the next round's prefetch target
  }
  cp_async_wait_all();
}

template <int NA, int NB>
cudaError_t launch_pair(const PairArgs& g, cudaStream_t st) {
  const int smem = (NA * NA + (NB > 1 ? NB * NB : 0) + 2 * g.bsz) * 8;
  auto k = pair_kernel<NA, NB>;
  int nsm = 0, occ = 0;
  if (cudaError_t e = kernel_setup(k, smem, THREADS, &nsm, &occ); e != cudaSuccess) return e;
  int64_t grid = static_cast<int64_t>(nsm) * occ;
  if (grid > g.nblk) grid = g.nblk;
  k<<<static_cast<unsigned>(grid), THREADS, smem, st>>>(g);
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
static_assert((40 * 40 * 2 + 2 * kBlockTarget) * 8 <= 227 * 1024,
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
    while (c * 2 * grp <= target && P % (c * 2) == 0) c *= 2;
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
