// K1 (TMA-staged): the strided-batched FP64 DMMA GEMM of gemm.cu with its
// operand tiles staged by the Tensor Memory Accelerator.
//
//   C[b] = alpha * A[b] * B[b] + beta * C[b]      (column-major, "NN")
//
// for the mode products of tsylv::mode_multiply (reference
// tensor.hpp:187-231 -> blas.hpp:25-41).  Same CTA tile as the cp.async
// kernel (64 x 64 x 16, four warps of 32x32 DMMA patches, up to four CTAs per
// SM), but:
//   * one elected thread issues `cp.async.bulk.tensor` boxes (SASS UTMALDG)
//     into a ring of stages guarded by full/empty mbarriers: no per-thread
//     copy addressing, no __syncthreads in the k loop, edges zero-filled by
//     the tensor maps (one kernel for interior and edge tiles);
//   * the stages are dense 128-byte rows written with SWIZZLE_128B: A as four
//     boxes of 16 (m) x 16 (k), B as one box of 16 (k) x 64 (n).  A 16-byte
//     chunk c of row r lands at chunk c ^ (r & 7).  The four k of one DMMA
//     step are taken as {0,1,4,5} (+2 for odd steps, +8 for the upper half) —
//     the contraction order is free as long as A and B agree — so that the
//     32 lanes of every fragment load hit each bank pair exactly twice, the
//     minimum for 64-bit shared loads (conflict-free without padding).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "gemm.h"
#include "tma.h"
#include "util.h"

namespace tsg {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int kThreads = 128;
constexpr int kStageDoubles = (BM * BK + BK * BN);   // 2048 doubles = 16 KB
constexpr int kStageBytes = kStageDoubles * 8;

template <int STAGES>
constexpr int tma_smem_bytes() {
  return STAGES * kStageBytes + 1024 /* alignment slack */ + 2 * STAGES * 8;
}

TSG_DEVINL void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

template <int STAGES, bool EARLY>
__global__ void __launch_bounds__(kThreads, 4)
dgemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                 GemmArgs g) {
  extern __shared__ uint8_t raw[];
  const uint32_t pad = (1024u - (smem_u32(raw) & 1023u)) & 1023u;
  double* smem = reinterpret_cast<double*>(raw + pad);
  uint64_t* full = reinterpret_cast<uint64_t*>(raw + pad + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int gq = lane >> 2, tq = lane & 3;

  // flattened grid: m-tile fastest (B-panel reuse in L2), then n-tile, batch
  const int64_t tiles_m = (g.M + BM - 1) / BM;
  const int64_t tiles_n = (g.N + BN - 1) / BN;
  const int64_t bid = g.drev ? static_cast<int64_t>(gridDim.x) - 1 - blockIdx.x : blockIdx.x;
  const int64_t mt = bid % tiles_m, nt = (bid / tiles_m) % tiles_n;
  const int m0 = static_cast<int>(mt) * BM, n0 = static_cast<int>(nt) * BN;
  int64_t bt = bid / (tiles_m * tiles_n);
  if (g.pflags && g.pdesc) bt = g.batch - 1 - bt;
  const int ba = g.sA ? static_cast<int>(bt) : 0, bb = g.sB ? static_cast<int>(bt) : 0;

  const int nk = (g.K + BK - 1) / BK;
  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    double* sa = smem + s * kStageDoubles;
    mbar_expect_tx(full + s, kStageBytes);
#pragma unroll
    for (int i = 0; i < BM / 16; ++i) tma_load_3d(sa + i * 256, &mapA, m0 + 16 * i, kt * BK, ba, full + s);
    tma_load_3d(sa + BM * BK, &mapB, kt * BK, n0, bb, full + s);
  };
  auto issue_first = [&]() {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s)
      if (s < nk) issue(s);
  };
  if (tid == 0) {
    if (EARLY) {
      prefetch_tmap(&mapA);
      prefetch_tmap(&mapB);
    }
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kThreads / 32);
    }
    mbar_fence_init();
    if (EARLY && !g.pflags) {
      // the first stages are in flight before the other warps get here
      if (!g.nowait) pdl_wait();
      issue_first();
    }
  }
  __syncthreads();
  if (!g.pflags && !g.nowait) pdl_wait();
  pdl_trigger();
  if (g.pflags) {
    // Slab chain (consumer): this batch reads the producer's columns
    // [bt * pcpb, (bt + 1) * pcpb): acquire the done flags of those tiles
    // instead of waiting for the whole producer grid (see gemm.h).
    const int c0 = static_cast<int>(bt * g.pcpb / g.pbn);
    const int c1 = static_cast<int>(((bt + 1) * g.pcpb - 1) / g.pbn);
    const int cnt = (c1 - c0 + 1) * g.ptm;
    for (int i = tid; i < cnt; i += kThreads) {
      const int* f = g.pflags + (i % g.ptm) + static_cast<int64_t>(c0 + i / g.ptm) * g.ptm;
      while (ld_acquire(f) != g.pepoch) __nanosleep(128);
    }
    __threadfence();
    fence_proxy_async();   // the TMA (async proxy) reads what the flags published
    __syncthreads();
  }
  if (tid == 0 && (!EARLY || g.pflags)) issue_first();

  // Swizzled fragment addresses (doubles, relative to the stage).
  const int kb = (tq & 1) + ((tq >> 1) << 2);   // 0, 1, 4, 5
  const int baseA = wm * 512 + kb * 16 + ((((gq >> 1) ^ kb)) << 1) + (gq & 1);
  const int baseB = BM * BK + (wn * 32 + gq) * 16 + ((((kb >> 1) ^ gq)) << 1) + (kb & 1);
  int aA[4], aB[4];
#pragma unroll
  for (int v = 0; v < 4; ++v) aA[v] = baseA ^ (v << 2);             // chunk ^ {0, 2, 4, 6}
#pragma unroll
  for (int s = 0; s < 4; ++s) aB[s] = baseB ^ (((s & 1) | ((s >> 1) << 2)) << 1);

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < nk; ++kt) {
    const int st = kt % STAGES;
    if (tid == 0) {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) {
        // stage of tile kt - 1: every warp has released it (or it is fresh)
        if (nxt >= STAGES) mbar_wait(empty + nxt % STAGES, ((nxt / STAGES) - 1) & 1);
        issue(nxt);
      }
    }
    mbar_wait(full + st, (kt / STAGES) & 1);
    const double* sp = smem + st * kStageDoubles;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        af[i] = sp[aA[((i & 1) << 1) ^ (s & 1)] + (i >> 1) * 256 + (s & 1) * 32 + (s >> 1) * 128];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = sp[aB[s] + j * 128];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
  }

  // Epilogue: C = alpha*acc + beta*C (beta == 0 never reads C).
  double* __restrict__ C = g.C + bt * g.sC;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + gq;
    if (row >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * 32 + j * 8 + 2 * tq + h;
        if (col >= g.N) continue;
        double* p = C + static_cast<int64_t>(col) * g.ldc + row;
        const double v = g.alpha * acc[i][j][h];
        *p = (g.beta == 0.0) ? v : v + g.beta * *p;
      }
    }
  }
  if (g.dflags) {   // slab chain (producer): done flag of this tile after all its stores
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(g.dflags + mt + nt * tiles_m, g.depoch);
    }
  }
}

int tma_variant() {
  // development A/B (TSG_GEMM_TMA): 1 = three stages (four CTAs per SM),
  // 2 = the same with the first stages issued ahead of the block barrier,
  // 4 = four stages (three CTAs per SM)
  static const int n = [] {
    const char* e = std::getenv("TSG_GEMM_TMA");
    const int v = e ? std::atoi(e) : 1;
    return (v == 2 || v == 4) ? v : 1;
  }();
  return n;
}

template <int STAGES, bool EARLY>
cudaError_t launch_tma(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& g, unsigned tiles,
                       cudaStream_t st) {
  auto k = dgemm_tma_kernel<STAGES, EARLY>;
  if (g.pdl) {
    if (cudaError_t e = launch_pdl(k, tiles, kThreads, tma_smem_bytes<STAGES>(), st, ma, mb, g); e != cudaSuccess)
      return e;
  } else {
    k<<<tiles, kThreads, tma_smem_bytes<STAGES>(), st>>>(ma, mb, g);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t gemm_tma_prepare() {
  int nsm = 0, occ = 0;
  cudaError_t e = kernel_setup(dgemm_tma_kernel<3, false>, tma_smem_bytes<3>(), kThreads, &nsm, &occ);
  if (e == cudaSuccess) e = kernel_setup(dgemm_tma_kernel<3, true>, tma_smem_bytes<3>(), kThreads, &nsm, &occ);
  if (e == cudaSuccess) e = kernel_setup(dgemm_tma_kernel<4, false>, tma_smem_bytes<4>(), kThreads, &nsm, &occ);
  return e;
}

bool gemm_tma_ok(const GemmArgs& g) {
  if (g.wflags) return false;   // the gated back transform of the tile-DAG path stays on gemm.cu
  if (g.M < 1 || g.N < 1 || g.K < 1 || g.batch < 1) return false;
  if ((g.lda | g.ldb) & 1) return false;
  if (g.batch > 1 && ((g.sA | g.sB) & 1)) return false;
  if ((reinterpret_cast<uintptr_t>(g.A) | reinterpret_cast<uintptr_t>(g.B)) & 15) return false;
  if (g.lda < g.M || g.ldb < g.K) return false;
  const int64_t lim = int64_t{1} << 36;   // tensor-map strides are < 2^40 bytes
  if (g.lda >= lim || g.ldb >= lim || g.sA >= lim || g.sB >= lim || g.batch > 0x7fffffffLL) return false;
  return true;
}

cudaError_t dgemm_nn_tma(const GemmArgs& g, cudaStream_t st) {
  const int64_t tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN) * g.batch;
  if (tiles <= 0) return cudaSuccess;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidValue;
  CUtensorMap ma, mb;
  {
    const uint64_t dims[3] = {static_cast<uint64_t>(g.M), static_cast<uint64_t>(g.K),
                              static_cast<uint64_t>(g.sA ? g.batch : 1)};
    const uint64_t str[2] = {static_cast<uint64_t>(g.lda) * 8,
                             static_cast<uint64_t>(g.sA ? g.sA : g.lda * g.K) * 8};
    const uint32_t box[3] = {16, BK, 1};
    if (!encode_tmap_f64_strided(&ma, g.A, 3, dims, str, box, true)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[3] = {static_cast<uint64_t>(g.K), static_cast<uint64_t>(g.N),
                              static_cast<uint64_t>(g.sB ? g.batch : 1)};
    const uint64_t str[2] = {static_cast<uint64_t>(g.ldb) * 8,
                             static_cast<uint64_t>(g.sB ? g.sB : g.ldb * g.N) * 8};
    const uint32_t box[3] = {BK, BN, 1};
    if (!encode_tmap_f64_strided(&mb, g.B, 3, dims, str, box, true)) return cudaErrorInvalidValue;
  }
  if (cudaError_t e = gemm_tma_prepare(); e != cudaSuccess) return e;
  const unsigned nt = static_cast<unsigned>(tiles);
  switch (tma_variant()) {
    case 4: return launch_tma<4, false>(ma, mb, g, nt, st);
    case 2: return launch_tma<3, true>(ma, mb, g, nt, st);
    default: return launch_tma<3, false>(ma, mb, g, nt, st);
  }
}

}  // namespace tsg
