// K1/K2: strided-batched FP64 GEMM on DMMA tensor cores (sm_100a).
//
// Replaces the dgemm_ calls issued by tsylv::mode_multiply
// (reference tensor.hpp:187-231 -> blas.hpp:25-41) for the forward/back
// Schur-basis transforms, and the in-place window updates of the recursion
// (laplace.hpp:147 `b1 -= mode_multiply(x2, A12, mu)`), as
//
//   C[b] = alpha * A[b] * B[b] + beta * C[b]      (column-major, "NN")
//
// with one batch index b (middle-mode slabs: tensor.hpp:218-229).  Every
// mode product maps onto it with no transpose copies: mode 0 is
// Y_(0) = A X_(0) (A small, B = the tensor), modes m > 0 are per-slab
// Y_slab = X_slab A^T (A = the tensor slab, B = the coefficient transposed
// on the host once).
//
// This file: the cp.async kernel (narrow shapes, misaligned operands, the
// tile-flag-gated back transform); products with both extents >= 64 go to
// the TMA-staged kernel of gemm_tma.cu by default.
//
// Design: CTA tile BM x BN x 16, 3-stage cp.async ring (L2-only .cg 16 B
// copies, zero-fill at the edges), 8 warps each owning a WM x WN patch of
// 8x8 DMMA accumulators in registers.  Shared-memory leading dimensions are
// padded to 4 (mod 16) doubles so that every half-warp fragment load hits 16
// distinct 8-byte bank pairs (conflict-free LDS.64).
#include <mutex>
#include <set>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "gemm.h"
#include "util.h"

namespace tsg {

namespace {

#ifndef TSG_GEMM_BK
#define TSG_GEMM_BK 16
#endif
constexpr int BK = TSG_GEMM_BK;
#ifndef TSG_GEMM_STAGES
#define TSG_GEMM_STAGES 3
#endif
constexpr int kStages = TSG_GEMM_STAGES;

template <int BM, int BN>
struct GemmSmem {
  static constexpr int LDA = BM + 4;   // A stage: [BK][LDA] (m fastest)
  static constexpr int LDB = BK + 4;   // B stage: [BN][LDB] (k fastest)
  static constexpr int A_ELEMS = BK * LDA;
  static constexpr int B_ELEMS = BN * LDB;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr int BYTES = kStages * STAGE * 8;
};

// Tile of this CTA and the cross-kernel waits every GEMM kernel shares.
// Flattened grid: m-tile fastest (B-panel reuse in L2), then n-tile, batch.
// Programmatic launches wait for the producer of A/B (pdl_wait), except the
// gated transforms, which acquire tile / slab flags instead; every grid
// then lets the next kernel's CTAs be scheduled as it drains.
template <int BM, int BN, int NT>
TSG_DEVINL void gemm_prologue(const GemmArgs& g, int tid, int64_t& mt, int64_t& nt, int64_t& bt,
                              int64_t& tiles_m) {
  const int64_t bid = g.drev ? static_cast<int64_t>(gridDim.x) - 1 - blockIdx.x : blockIdx.x;
  tiles_m = (g.M + BM - 1) / BM;
  const int64_t tiles_n = (g.N + BN - 1) / BN;
  mt = bid % tiles_m;
  nt = (bid / tiles_m) % tiles_n;
  bt = bid / (tiles_m * tiles_n);
  if (!g.wflags && !g.pflags && !g.nowait) pdl_wait();
  pdl_trigger();
  if (g.pflags) {
    if (g.pdesc) bt = g.batch - 1 - bt;
    const int c0 = static_cast<int>(bt * g.pcpb / g.pbn);
    const int c1 = static_cast<int>(((bt + 1) * g.pcpb - 1) / g.pbn);
    const int cnt = (c1 - c0 + 1) * g.ptm;
    for (int i = tid; i < cnt; i += NT) {
      const int* f = g.pflags + (i % g.ptm) + static_cast<int64_t>(c0 + i / g.ptm) * g.ptm;
      while (ld_acquire(f) != g.pepoch) __nanosleep(128);
    }
    __threadfence();
    __syncthreads();
  }
  if (g.wflags) {
    // Gated back transform: the solve releases the last columns first.
    nt = tiles_n - 1 - nt;
    const int c0 = static_cast<int>(nt * BN) / kWaitCols;
    const int c1 = min(g.wgroups, static_cast<int>((nt * BN + BN + kWaitCols - 1) / kWaitCols));
    for (int i = g.woff[c0] + tid; i < g.woff[c1]; i += NT) {
      const int* f = g.wflags + g.wids[i];
      while (ld_acquire(f) != g.wepoch) __nanosleep(256);
    }
    __threadfence();
    __syncthreads();
  }
}

// Done flag of a producer CTA tile (slab chain), after all its stores.
TSG_DEVINL void gemm_done(const GemmArgs& g, int tid, int64_t mt, int64_t nt, int64_t tiles_m) {
  if (g.dflags) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(g.dflags + mt + nt * tiles_m, g.depoch);
    }
  }
}

#ifndef TSG_GEMM_MINB
#define TSG_GEMM_MINB 1
#endif
template <int BM, int BN, int WM, int WN, bool VEC, bool FAST = false>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32,
                                  (FAST && (BM / WM) * (BN / WN) == 4) ? 4 : TSG_GEMM_MINB)
dgemm_nn_kernel(GemmArgs g) {
  using S = GemmSmem<BM, BN>;
  constexpr int NWM = BM / WM;              // warps along M
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  constexpr int FM = WM / 8, FN = WN / 8;   // 8x8 fragments per warp
  extern __shared__ __align__(16) double smem[];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % NWM, wn = warp / NWM;
  const int gq = lane >> 2, tq = lane & 3;

  int64_t mt, nt, bt, tiles_m;
  gemm_prologue<BM, BN, NT>(g, tid, mt, nt, bt, tiles_m);
  const int m0 = static_cast<int>(mt * BM), n0 = static_cast<int>(nt * BN);

  const double* __restrict__ A = g.A + bt * g.sA;
  const double* __restrict__ B = g.B + bt * g.sB;
  double* __restrict__ C = g.C + bt * g.sC;

  auto load_stage = [&](int stage, int k0) {
    double* sa = smem + stage * S::STAGE;
    double* sb = sa + S::A_ELEMS;
    if (VEC) {
      // A: BK columns of BM contiguous doubles -> 16-byte chunks.
      constexpr int ACH = BK * BM / 2;
      for (int c = tid; c < ACH; c += NT) {
        const int kk = c / (BM / 2), mm = (c % (BM / 2)) * 2;
        const int gm = m0 + mm, gk = k0 + kk;
        int bytes = 0;
        const double* src = A;
        if (gk < g.K && gm < g.M) {
          bytes = (g.M - gm >= 2) ? 16 : 8;
          src = A + static_cast<int64_t>(gk) * g.lda + gm;
        }
        cp_async16(sa + kk * S::LDA + mm, src, bytes);
      }
      // B: BN columns of BK contiguous doubles.
      constexpr int BCH = BN * BK / 2;
      for (int c = tid; c < BCH; c += NT) {
        const int nn = c / (BK / 2), kk = (c % (BK / 2)) * 2;
        const int gn = n0 + nn, gk = k0 + kk;
        int bytes = 0;
        const double* src = B;
        if (gn < g.N && gk < g.K) {
          bytes = (g.K - gk >= 2) ? 16 : 8;
          src = B + static_cast<int64_t>(gn) * g.ldb + gk;
        }
        cp_async16(sb + nn * S::LDB + kk, src, bytes);
      }
    } else {
      for (int c = tid; c < BK * BM; c += NT) {
        const int kk = c / BM, mm = c % BM;
        const int gm = m0 + mm, gk = k0 + kk;
        const bool ok = gk < g.K && gm < g.M;
        cp_async8(sa + kk * S::LDA + mm,
                  ok ? A + static_cast<int64_t>(gk) * g.lda + gm : A, ok ? 8 : 0);
      }
      for (int c = tid; c < BN * BK; c += NT) {
        const int nn = c / BK, kk = c % BK;
        const int gn = n0 + nn, gk = k0 + kk;
        const bool ok = gn < g.N && gk < g.K;
        cp_async8(sb + nn * S::LDB + kk,
                  ok ? B + static_cast<int64_t>(gn) * g.ldb + gk : B, ok ? 8 : 0);
      }
    }
  };

  // Interior tiles (no M/N edge, K a multiple of BK, 16-byte aligned): the
  // per-thread copy sources are fixed pointers advanced by BK per k-tile.
  constexpr int ACH = BK * BM / 2, BCH = BN * BK / 2;
  constexpr int NA = (ACH + NT - 1) / NT, NB = (BCH + NT - 1) / NT;
  // FAST instantiations are launched only when every tile is interior
  constexpr bool interior = FAST;
  // 32-bit per-thread source offsets (the operands' tile panels are small)
  const double* A0 = A + m0;
  const double* B0 = B + static_cast<int64_t>(n0) * g.ldb;
  int ga[NA], gb[NB], oa[NA], ob[NB];
  if constexpr (FAST) {
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const int c = tid + i * NT;
      const int kk = c / (BM / 2), mm = (c % (BM / 2)) * 2;
      ga[i] = kk * static_cast<int>(g.lda) + mm;
      oa[i] = kk * S::LDA + mm;
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int c = tid + i * NT;
      const int nn = c / (BK / 2), kk = (c % (BK / 2)) * 2;
      gb[i] = nn * static_cast<int>(g.ldb) + kk;
      ob[i] = nn * S::LDB + kk;
    }
  }
  const int64_t astep = static_cast<int64_t>(BK) * g.lda;
  auto load_fast = [&](int stage, int kt) {
    double* sa = smem + stage * S::STAGE;
    double* sb = sa + S::A_ELEMS;
    const double* ak = A0 + kt * astep;
    const double* bk = B0 + kt * BK;
#pragma unroll
    for (int i = 0; i < NA; ++i)
      if (ACH % NT == 0 || tid + i * NT < ACH) cp_async16(sa + oa[i], ak + ga[i], 16);
#pragma unroll
    for (int i = 0; i < NB; ++i)
      if (BCH % NT == 0 || tid + i * NT < BCH) cp_async16(sb + ob[i], bk + gb[i], 16);
  };

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (g.K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) {
      if constexpr (interior) load_fast(s, s);
      else load_stage(s, s * BK);
    }
    cp_async_commit();
  }

  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int nxt = kt + kStages - 1;
      if (nxt < nk) {
        if constexpr (interior) load_fast(nxt % kStages, nxt);
        else load_stage(nxt % kStages, nxt * BK);
      }
      cp_async_commit();
    }
    const double* sa = smem + (kt % kStages) * S::STAGE;
    const double* sb = sa + S::A_ELEMS;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i)
        af[i] = sa[(k4 + tq) * S::LDA + wm * WM + i * 8 + gq];
#pragma unroll
      for (int j = 0; j < FN; ++j)
        bf[j] = sb[(wn * WN + j * 8 + gq) * S::LDB + k4 + tq];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait_all();

  // Epilogue: C = alpha*acc + beta*C (beta == 0 never reads C).
#pragma unroll
  for (int i = 0; i < FM; ++i) {
    const int row = m0 + wm * WM + i * 8 + gq;
    if (row >= g.M) continue;
#pragma unroll
    for (int j = 0; j < FN; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * WN + j * 8 + 2 * tq + h;
        if (col >= g.N) continue;
        double* p = C + static_cast<int64_t>(col) * g.ldc + row;
        const double v = g.alpha * acc[i][j][h];
        *p = (g.beta == 0.0) ? v : v + g.beta * *p;
      }
    }
  }
  gemm_done(g, tid, mt, nt, tiles_m);
}

template <typename K>
void launch_k(K k, unsigned grid, int threads, int smem, const GemmArgs& g, cudaStream_t st) {
  if (!g.pdl) {
    k<<<grid, threads, smem, st>>>(g);
    return;
  }
  launch_pdl(k, grid, threads, smem, st, g);
}

template <int BM, int BN, int WM, int WN>
cudaError_t launch_cfg(const GemmArgs& g, cudaStream_t st) {
  using S = GemmSmem<BM, BN>;
  const int64_t tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN) * g.batch;
  if (tiles <= 0) return cudaSuccess;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidValue;
  const bool vec = (g.lda % 2 == 0) && (g.ldb % 2 == 0) && (g.sA % 2 == 0) && (g.sB % 2 == 0) &&
                   ((reinterpret_cast<uintptr_t>(g.A) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(g.B) & 15) == 0);
  const bool all_interior = vec && g.M % BM == 0 && g.N % BN == 0 && g.K % BK == 0 &&
                            g.lda * BK < (int64_t{1} << 30) && g.ldb * BN < (int64_t{1} << 30);
  if (all_interior) {
    auto k = dgemm_nn_kernel<BM, BN, WM, WN, true, true>;
    int nsm = 0, occ = 0;
    if (cudaError_t e = kernel_setup(k, S::BYTES, (BM / WM) * (BN / WN) * 32, &nsm, &occ); e != cudaSuccess) return e;
    launch_k(k, static_cast<unsigned>(tiles), (BM / WM) * (BN / WN) * 32, S::BYTES, g, st);
  } else if (vec) {
    auto k = dgemm_nn_kernel<BM, BN, WM, WN, true>;
    int nsm = 0, occ = 0;
    if (cudaError_t e = kernel_setup(k, S::BYTES, (BM / WM) * (BN / WN) * 32, &nsm, &occ); e != cudaSuccess) return e;
    launch_k(k, static_cast<unsigned>(tiles), (BM / WM) * (BN / WN) * 32, S::BYTES, g, st);
  } else {
    auto k = dgemm_nn_kernel<BM, BN, WM, WN, false>;
    int nsm = 0, occ = 0;
    if (cudaError_t e = kernel_setup(k, S::BYTES, (BM / WM) * (BN / WN) * 32, &nsm, &occ); e != cudaSuccess) return e;
    launch_k(k, static_cast<unsigned>(tiles), (BM / WM) * (BN / WN) * 32, S::BYTES, g, st);
  }
  return cudaGetLastError();
}

}  // namespace

void gemm_tile_shape(int M, int N, int* bm, int* bn) {
  // mirrors the default dispatch of dgemm_nn below
  if (const char* e = std::getenv("TSG_GEMM_CFG"); e && std::atoi(e) != 0) {
    *bm = *bn = 0;
    return;
  }
  if (M >= 64 && N >= 64) *bm = 64, *bn = 64;
  else if (N <= 64 && M >= 128) *bm = 128, *bn = 64;
  else if (M <= 64 && N >= 128) *bm = 64, *bn = 128;
  else if (M <= 64 && N <= 64) *bm = 64, *bn = 64;
  else *bm = 128, *bn = 128;
}

// Shared-memory attributes of every kernel the default dispatch can pick,
// set once up front: a cudaFuncSetAttribute between two launches of a
// programmatic-dependent pair (first use of an instantiation) serialises
// them, and the trailing-cube grid waits on its dependent GEMM.
template <int BM, int BN, int WM, int WN>
cudaError_t set_attrs() {
  const int bytes = GemmSmem<BM, BN>::BYTES, threads = (BM / WM) * (BN / WN) * 32;
  int nsm = 0, occ = 0;
  cudaError_t e = kernel_setup(dgemm_nn_kernel<BM, BN, WM, WN, true, true>, bytes, threads, &nsm, &occ);
  if (e == cudaSuccess) e = kernel_setup(dgemm_nn_kernel<BM, BN, WM, WN, true>, bytes, threads, &nsm, &occ);
  if (e == cudaSuccess) e = kernel_setup(dgemm_nn_kernel<BM, BN, WM, WN, false>, bytes, threads, &nsm, &occ);
  return e;
}

// per device (kernel_setup caches per (kernel, device); this only saves the walk)
cudaError_t gemm_prepare() {
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (done.count(dev)) return cudaSuccess;
  }
  cudaError_t e = set_attrs<64, 64, 32, 32>();
  if (e == cudaSuccess) e = set_attrs<128, 64, 32, 32>();
  if (e == cudaSuccess) e = set_attrs<64, 128, 32, 32>();
  if (e == cudaSuccess) e = set_attrs<64, 64, 32, 16>();
  if (e == cudaSuccess) e = set_attrs<128, 128, 64, 32>();
  if (e == cudaSuccess) e = set_attrs<128, 128, 32, 32>();
  if (e == cudaSuccess) e = set_attrs<128, 128, 32, 64>();
  if (e == cudaSuccess) e = set_attrs<128, 128, 64, 64>();
  if (e == cudaSuccess) e = set_attrs<128, 64, 64, 16>();
  if (e == cudaSuccess) e = gemm_tma_prepare();
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  done.insert(dev);
  return cudaSuccess;
}

cudaError_t dgemm_nn(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return cudaSuccess;
  if (cudaError_t e = gemm_prepare(); e != cudaSuccess) return e;
  static const int cfg = [] {
    const char* e = std::getenv("TSG_GEMM_CFG");
    return e ? std::atoi(e) : 0;
  }();
  // Default for both extents >= 64: the TMA-staged 64x64 kernel
  // (gemm_tma.cu; C4 transforms 34.9 -> 35.6 TF/s, profiles/r02l_*);
  // TSG_GEMM_TMA=0 keeps the cp.async kernel below (development A/B).  The
  // gated back transform of the tile-DAG path (wflags) stays on cp.async.
  static const int tma = [] {
    const char* e = std::getenv("TSG_GEMM_TMA");
    return e ? std::atoi(e) : 1;
  }();
  if (tma && cfg == 0 && g.M >= 64 && g.N >= 64 && gemm_tma_ok(g)) return dgemm_nn_tma(g, st);
  if (cfg == 1 && g.M >= 128 && g.N >= 64) return launch_cfg<128, 64, 32, 32>(g, st);   // 8 warps, 2 CTA/SM
  if (cfg == 2 && g.M >= 128 && g.N >= 128) return launch_cfg<128, 128, 32, 32>(g, st); // 16 warps
  if (cfg == 3 && g.M >= 128 && g.N >= 128) return launch_cfg<128, 128, 32, 64>(g, st); // 8 warps 32x64
  if (cfg == 4 && g.M >= 64 && g.N >= 128) return launch_cfg<64, 128, 32, 32>(g, st);   // 8 warps
  if (cfg == 5 && g.M >= 128 && g.N >= 128) return launch_cfg<128, 128, 64, 64>(g, st); // 4 warps
  if (cfg == 6 && g.M >= 64 && g.N >= 64) return launch_cfg<64, 64, 32, 32>(g, st);      // 4 warps
  if (cfg == 7 && g.M >= 128 && g.N >= 64) return launch_cfg<128, 64, 64, 16>(g, st);    // 8 warps
  // Default: 64x64 CTA tiles of four 32x32-DMMA warps (up to 4 CTAs/SM);
  // measured best on the C2/C4 transforms (29-32 TF/s vs 24-25 for 128x128
  // with one CTA per SM, profiles/r01_gemm_configs.log).
  if (g.M >= 64 && g.N >= 64) return launch_cfg<64, 64, 32, 32>(g, st);
  // Small-N slabs (middle-mode transforms with n_m < 64) / small-M.
  if (g.N <= 64 && g.M >= 128) return launch_cfg<128, 64, 32, 32>(g, st);
  if (g.M <= 64 && g.N >= 128) return launch_cfg<64, 128, 32, 32>(g, st);
  if (g.M <= 64 && g.N <= 64) return launch_cfg<64, 64, 32, 16>(g, st);
  return launch_cfg<128, 128, 64, 32>(g, st);
}

}  // namespace tsg

namespace tsg {

cudaError_t mode_product(const double* X, double* Y, int d, const int* dims, int mode,
                         const double* A, const double* At, int r, double alpha, double beta,
                         cudaStream_t st, double* flops, const GemmArgs* gate) {
  int64_t P = 1, Q = 1;
  for (int v = 0; v < mode; ++v) P *= dims[v];
  for (int v = mode + 1; v < d; ++v) Q *= dims[v];
  const int n = dims[mode];
  GemmArgs g{};
  g.alpha = alpha;
  g.beta = beta;
  if (mode == 0) {
    // Y_(0) (r x Q) = A (r x n) * X_(0) (n x Q)      (tensor.hpp:203-210)
    g.A = A;
    g.B = X;
    g.C = Y;
    g.M = r;
    g.N = static_cast<int>(Q);
    g.K = n;
    g.lda = r;
    g.ldb = n;
    g.ldc = r;
    g.sA = g.sB = g.sC = 0;
    g.batch = 1;
    if (Q > 0x7fffffffLL) return cudaErrorInvalidValue;
    if (gate) {
      g.wflags = gate->wflags;
      g.woff = gate->woff;
      g.wids = gate->wids;
      g.wepoch = gate->wepoch;
      g.wgroups = gate->wgroups;
    }
  } else {
    // per slab q: Y_q (P x r) = X_q (P x n) * A^T (n x r)  (tensor.hpp:211-229)
    if (P > 0x7fffffffLL) return cudaErrorInvalidValue;
    g.A = X;
    g.B = At;
    g.C = Y;
    g.M = static_cast<int>(P);
    g.N = r;
    g.K = n;
    g.lda = P;
    g.ldb = n;
    g.ldc = P;
    g.sA = P * n;
    g.sB = 0;
    g.sC = P * r;
    g.batch = Q;
  }
  if (gate) {
    g.pdl = gate->pdl;
    g.nowait = gate->nowait;
    if (g.batch == 1) {
      g.dflags = gate->dflags;
      g.depoch = gate->depoch;
      g.drev = gate->drev;
    } else {
      g.pflags = gate->pflags;
      g.pepoch = gate->pepoch;
      g.ptm = gate->ptm;
      g.pbn = gate->pbn;
      g.pcpb = gate->pcpb;
      g.pdesc = gate->pdesc;
    }
  }
  if (flops) *flops += 2.0 * static_cast<double>(P) * Q * n * r;
  return dgemm_nn(g, st);
}

}  // namespace tsg
