// Order-3 Laplace solve over 16^3 tiles with TMA-staged operands (C2, C4).
//
// Same dataflow as solve_lap3.cu (tiles in topological hyperplane order from
// an atomic queue, left-looking updates from later tiles, release flags),
// rebuilt around the two costs that bound the 8^3 kernel:
//   * update traffic: every B element loaded for the left-looking update
//     feeds one row block per tile extent, so 16-row tiles halve the L2
//     traffic of sum_m T_m[t, later] x_m X(later) (24 N vs 48 N doubles);
//   * memory-level parallelism: one producer warp streams the update
//     operand as 16x16x16 boxes of X (cp.async.bulk.tensor, padded to
//     20x17x16 = 43.5 KB for conflict-free fragment loads) through an
//     mbarrier ring (two stages here, three in the decoupled kernel below,
//     which is the default), so the eight consumer warps only issue DMMA and
//     shared-memory fragment loads (no register-bound load batches).
// The base case block-diagonalises the tile over the reals: with V_m the real
// eigenvector basis of the tile's diagonal Schur block (1x1 cells keep their
// eigenvector, 2x2 cells take [Re v, Im v]),
//   y = x x_0 V0^-1 x_1 V1^-1 x_2 V2^-1,  cell solves (<= 8 unknowns each,
//   closed form, cell_solve16),  x = y x_m V_m:
// six real 16x16x256 DMMA GEMMs (this kernel: the ring as the work tile;
// the decoupled kernel: in place).  Plans choose these kernels only when every
// tile's bases are well conditioned (tsg_plan: vcond product <= kDiagCond).
// One CTA (8 consumer + 1 producer warps) per SM.
// Reference: lap_rec / lap_base (laplace.hpp:99-153), mode_multiply update
// (laplace.hpp:147), block_back_substitution (kernels.hpp:179-261).
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "solve.h"
#include "tma.h"
#include "util.h"

namespace tsg {
namespace {

#ifndef L16_PROF
#define L16_PROF 0
#endif
#ifndef L16_ORDER_AB
#define L16_ORDER_AB 1  // decoupled kernel: far chunks of tiles >= t+3 first, then the t+2 rows of every mode
#endif
#ifndef L16_TRACE2
#define L16_TRACE2 0  // development: claim / far-done / chunks-done times per tile (TSG_TRACE)
#endif

constexpr int E = 16, EE = 256, TT = 4096;
constexpr int CW = 8;                 // consumer warps
constexpr int THREADS = (CW + 1) * 32;
#ifndef L16_NST
#define L16_NST 2
#endif
#ifndef L16_BY
#define L16_BY 17
#endif
#ifndef L16_BX
#define L16_BX 20
#endif
constexpr int NSR = L16_NST;          // ring stages in the ring region
constexpr int NST = NSR + 1;          // + xi (free while the updates stream)
constexpr int VHS = kVhStride16;
// Shared tile layout = the TMA box layout: (x0, x1, x2) at x0 + S1 x1 + S2 x2.
// Boxes are 20 x 17 x 16: the inner start coordinate of an FP64 box must be
// even (16-byte aligned), so a box starts at c0 & ~1 and the 16 used
// elements sit at offset o = c0 & 1; the padded strides (20, 340 doubles)
// make every DMMA fragment load of the three modes bank-conflict free.
constexpr int BX = L16_BX, BY = L16_BY, BZ = 16;
constexpr int S1 = BX, S2 = BX * BY, TD = BX * BY * BZ;
constexpr int OFF_XR = 0, OFF_XI = TD, OFF_VH = 2 * TD, OFF_RING = OFF_VH + 3 * VHS;
constexpr int DOUBLES = OFF_RING + NSR * TD;
constexpr int BYTES = DOUBLES * 8;
constexpr unsigned BOX_BYTES = TD * 8;
static_assert((OFF_RING * 8) % 128 == 0 && (TD * 8) % 128 == 0, "TMA destinations 128-byte aligned");
static_assert(NSR >= 2, "the ring doubles as the complex work tile (yr, yi)");

struct G16 {
  int64_t lt, gbase;
  int start[3], ext[3], tco[3];
  int nlo[3], flo[3];  // first rows of tiles t+1 and t+2 per mode (n_m when absent)
  int nch;             // chunks of this tile
  int done;            // decoupled kernel: no more tiles
  int nc[3];           // Schur cells (1x1 / 2x2) of the tile's diagonal blocks
  unsigned char cs[3][16], cz[3][16];
  unsigned ck[208];    // decoupled kernel: the tile's chunk list (pack_chunk), n_m <= 1024
};

TSG_DEVINL void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
TSG_DEVINL void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
TSG_DEVINL void consumers_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(CW * 32) : "memory"); }

// tile offset of mode-M row i, cross-section column n (the other two modes,
// first one fastest); also the layout of a 16^3 TMA box along mode M
template <int M>
TSG_DEVINL int addr16(int i, int n) {
  if (M == 0) return i + S1 * (n & (E - 1)) + S2 * (n >> 4);
  if (M == 1) return (n & (E - 1)) + S1 * i + S2 * (n >> 4);
  return (n & (E - 1)) + S1 * (n >> 4) + S2 * i;
}

// chunk c of the tile: mode, first row, end row (far ranges first, then the
// near tiles t+1), identical on the producer and the consumers.  Far ranges
// (tiles >= t+2) run top down, so the chunks of long-finished tiles go first
// and the t+2 rows, released last, come at the end of the group (the
// producer waits per chunk on the tile holding its first row).
struct Chunk {
  int m, k, kh, first;  // first: first chunk of its (mode, far/near) group
};
TSG_DEVINL Chunk chunk_of(const G16& g, const int* dims, int c) {
#pragma unroll
  for (int part = 0; part < 2; ++part)
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int lo = part == 0 ? g.flo[m] : g.nlo[m];
      const int hi = part == 0 ? dims[m] : g.flo[m];
      const int n = hi > lo ? (hi - lo + E - 1) / E : 0;
      if (c < n) {
        if (part == 0) {
          const int k = lo + E * (n - 1 - c);
          return Chunk{m, k, min(k + E, hi), c == 0};
        }
        return Chunk{m + 3, lo + E * c, hi, c == 0};
      }
      c -= n;
    }
  return Chunk{0, 0, 0, 0};
}

// chunk list entries: mode group (3 bits), first row, end row (12 bits
// each), first-of-group flag; built once per tile by the producer warp
TSG_DEVINL unsigned pack_chunk(const Chunk& c) {
  return static_cast<unsigned>(c.m) | (static_cast<unsigned>(c.k) << 3) | (static_cast<unsigned>(c.kh) << 15) |
         (static_cast<unsigned>(c.first) << 27);
}
TSG_DEVINL Chunk unpack_chunk(unsigned v) {
  return Chunk{static_cast<int>(v & 7u), static_cast<int>((v >> 3) & 4095u), static_cast<int>((v >> 15) & 4095u),
               static_cast<int>(v >> 27)};
}

// acc[rb][cb] += T_M[rows, k..k+15] * box(k, cols) for this warp's 4 column
// blocks (cross-section columns 32 w .. 32 w + 31), both 8-row blocks
// A fragments of a chunk: T_M[tile rows, k..k+15] (rows beyond the tensor
// clamp, columns >= kh give 0)
TSG_DEVINL void chunk_afrag(const SolveArgs& a, const G16& g, int m, int k, int kh, double (&af)[4][2]) {
  const int lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int n = a.dims[m];
  const double* Tm = a.T[m];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks)
#pragma unroll
    for (int rb = 0; rb < 2; ++rb) {
      const int kk = k + 4 * ks + tq;
      int row = g.start[m] + 8 * rb + gq;
      row = row < n ? row : n - 1;
      af[ks][rb] = kk < kh ? __ldg(Tm + row + static_cast<int64_t>(kk) * n) : 0.0;
    }
}

// acc[rb][cb] += A(16 rows x 16 k) * box(k, cols) for this warp's 4 column
// blocks (cross-section columns 32 w .. 32 w + 31), both 8-row blocks
template <int M>
TSG_DEVINL void chunk_dmma(const double* box, const double (&af)[4][2], double (&acc)[2][4][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) {
      const double b = box[addr16<M>(4 * ks + tq, 8 * (4 * warp + cb) + gq)];
#pragma unroll
      for (int rb = 0; rb < 2; ++rb) dmma(acc[rb][cb][0], acc[rb][cb][1], af[ks][rb], b);
    }
}

template <int M>
TSG_DEVINL void flush16(double* xr, const double (&acc)[2][4][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int rb = 0; rb < 2; ++rb)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int h = 0; h < 2; ++h) xr[addr16<M>(8 * rb + gq, 8 * (4 * warp + cb) + 2 * tq + h)] -= acc[rb][cb][h];
}

// one complex 16x16 mode product over the tile (out of place), optional
// fused division by mu = l0 + l1 + l2 (mode 2 only)
template <int M, bool CIN, bool COUT, bool DIV>
TSG_DEVINL bool cmode16(const double* sr, const double* si, double* dr, double* di, const double* Ar,
                        const double* Ai, const double* vh, const int* ext, double tiny) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  double cr[2][4][2], ci[2][4][2];
#pragma unroll
  for (int rb = 0; rb < 2; ++rb)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) cr[rb][cb][0] = cr[rb][cb][1] = ci[rb][cb][0] = ci[rb][cb][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int k = 4 * ks + tq;
    double ar[2], ai[2];
#pragma unroll
    for (int rb = 0; rb < 2; ++rb) {
      ar[rb] = Ar[E * (8 * rb + gq) + k];
      ai[rb] = Ai[E * (8 * rb + gq) + k];
    }
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) {
      const int n = 8 * (4 * warp + cb) + gq;
      const double br = sr[addr16<M>(k, n)];
      const double bi = CIN ? si[addr16<M>(k, n)] : 0.0;
#pragma unroll
      for (int rb = 0; rb < 2; ++rb) {
        dmma(cr[rb][cb][0], cr[rb][cb][1], ar[rb], br);
        if (COUT) dmma(ci[rb][cb][0], ci[rb][cb][1], ai[rb], br);
        if (CIN) {
          dmma(cr[rb][cb][0], cr[rb][cb][1], -ai[rb], bi);
          if (COUT) dmma(ci[rb][cb][0], ci[rb][cb][1], ar[rb], bi);
        }
      }
    }
  }
  bool sing = false;
  // every element of the warp's 32 cross-section columns is read (above)
  // and written (below) by this warp only: in place needs just this
  __syncwarp();
#pragma unroll
  for (int rb = 0; rb < 2; ++rb)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = 8 * rb + gq, n = 8 * (4 * warp + cb) + 2 * tq + h;
        double vr = cr[rb][cb][h], vi = ci[rb][cb][h];
        if (DIV) {  // M == 2: rows i2, columns (i0, i1)
          const int i0 = n & (E - 1), i1 = n >> 4;
          const double mr = vh[4 * EE + i0] + vh[VHS + 4 * EE + i1] + vh[2 * VHS + 4 * EE + row];
          const double mi = vh[4 * EE + E + i0] + vh[VHS + 4 * EE + E + i1] + vh[2 * VHS + 4 * EE + E + row];
          const double den = mr * mr + mi * mi;
          if (!(den > tiny * tiny)) {
            if (i0 < ext[0] && i1 < ext[1] && row < ext[2]) sing = true;
            vr = vi = 0.0;
          } else {
            const double inv = 1.0 / den;
            const double r = (cr[rb][cb][h] * mr + ci[rb][cb][h] * mi) * inv;
            vi = (ci[rb][cb][h] * mr - cr[rb][cb][h] * mi) * inv;
            vr = r;
          }
        }
        dr[addr16<M>(row, n)] = vr;
        if (COUT) di[addr16<M>(row, n)] = vi;
      }
  return sing;
}

// Block-diagonal Kronecker-sum solve of the transformed tile, in place: with
// V_m^-1 D_m V_m = B_m (1x1 alpha, 2x2 [[alpha, beta], [-beta, alpha]]) the
// system sum_m B_m x_m Y = R decouples into cells (one Schur cell per mode,
// <= 8 unknowns); on a cell, the pair modes are diagonalised by the fixed
// butterfly E = [[1, 1], [i, -i]] (eigenvalues alpha +- i beta), so
//   y = Re( E (x) E (x) E  diag(1 / mu)  E^-1 (x) E^-1 (x) E^-1  r ),
//   mu = sum_m alpha_m + i s_m beta_m.
TSG_DEVINL bool cell_solve16(double* y, const G16& g, const double* vh, double tiny) {
  const int nc0 = g.nc[0], nc1 = g.nc[1], nc2 = g.nc[2];
  const int ncell = nc0 * nc1 * nc2;
  bool sing = false;
  for (int q = threadIdx.x; q < ncell; q += CW * 32) {
    const int c[3] = {q % nc0, (q / nc0) % nc1, q / (nc0 * nc1)};
    int r[3], z[3];
    double al[3], be[3];
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      r[m] = g.cs[m][c[m]];
      z[m] = g.cz[m][c[m]];
      al[m] = vh[m * VHS + 2 * EE + r[m]];
      be[m] = z[m] == 2 ? vh[m * VHS + 2 * EE + E + r[m]] : 0.0;
    }
    const bool valid = r[0] < g.ext[0] && r[1] < g.ext[1] && r[2] < g.ext[2];
    double zr[8], zi[8];
#pragma unroll
    for (int idx = 0; idx < 8; ++idx) {
      const int a0 = idx & 1, a1 = (idx >> 1) & 1, a2 = idx >> 2;
      const bool in = a0 < z[0] && a1 < z[1] && a2 < z[2];
      zr[idx] = in ? y[(r[0] + a0) + S1 * (r[1] + a1) + S2 * (r[2] + a2)] : 0.0;
      zi[idx] = 0.0;
    }
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      if (z[m] != 2) continue;
      const int bit = 1 << m;
#pragma unroll
      for (int idx = 0; idx < 8; ++idx) {
        if (idx & bit) continue;
        const double ur = zr[idx], ui = zi[idx], vr = zr[idx | bit], vi = zi[idx | bit];
        zr[idx] = 0.5 * (ur + vi);
        zi[idx] = 0.5 * (ui - vr);
        zr[idx | bit] = 0.5 * (ur - vi);
        zi[idx | bit] = 0.5 * (ui + vr);
      }
    }
#pragma unroll
    for (int idx = 0; idx < 8; ++idx) {
      double mr = 0.0, mi = 0.0;
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        mr += al[m];
        mi += ((idx >> m) & 1) ? -be[m] : be[m];
      }
      const double den = mr * mr + mi * mi;
      if (!(den > tiny * tiny)) {
        if (valid) sing = true;
        zr[idx] = zi[idx] = 0.0;
      } else {
        const double inv = 1.0 / den;
        const double nr = (zr[idx] * mr + zi[idx] * mi) * inv;
        zi[idx] = (zi[idx] * mr - zr[idx] * mi) * inv;
        zr[idx] = nr;
      }
    }
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      if (z[m] != 2) continue;
      const int bit = 1 << m;
#pragma unroll
      for (int idx = 0; idx < 8; ++idx) {
        if (idx & bit) continue;
        const double ur = zr[idx], ui = zi[idx], vr = zr[idx | bit], vi = zi[idx | bit];
        zr[idx] = ur + vr;            // u + v
        zi[idx] = ui + vi;
        zr[idx | bit] = vi - ui;      // i (u - v)
        zi[idx | bit] = ur - vr;
      }
    }
#pragma unroll
    for (int idx = 0; idx < 8; ++idx) {
      const int a0 = idx & 1, a1 = (idx >> 1) & 1, a2 = idx >> 2;
      if (a0 < z[0] && a1 < z[1] && a2 < z[2])
        y[(r[0] + a0) + S1 * (r[1] + a1) + S2 * (r[2] + a2)] = zr[idx];
    }
  }
  return sing;
}

TSG_DEVINL void wait_tile(const SolveArgs& a, int64_t tile) {
  const int* f = a.flags + tile;
  unsigned ns = 32;
  while (ld_acquire(f) < a.epoch) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    solve_lap16_kernel(SolveArgs a, const __grid_constant__ CUtensorMap tmx) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) double smem[];
  __shared__ G16 g;
  __shared__ int s_tile;
  __shared__ __align__(8) uint64_t full[NST], empty[NST], bar_x, bar_v;
  double* xr = smem + OFF_XR;
  double* xi = smem + OFF_XI;
  double* vh = smem + OFF_VH;
  double* ring = smem + OFF_RING;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, CW);
    }
    mbar_init(&bar_x, 1);
    mbar_init(&bar_v, 1);
    mbar_fence_init();
  }
  __syncthreads();
  unsigned gch = 0;   // chunks consumed/produced so far (ring phases)
  unsigned tphase = 0;  // tiles processed (bar_x / bar_v phases)
  const int64_t mul[3] = {1, a.ntiles_mode[0], static_cast<int64_t>(a.ntiles_mode[0]) * a.ntiles_mode[1]};

  // optional per-phase cycle counters of consumer thread 0 (TSG_PROF):
  // 0 claim+geometry, 1 first box wait, 2 update chunks, 3 flush, 4 diag,
  // 5 scatter+release; producer thread: 6 flag waits, 7 ring waits
  unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tmark = clock64();
  auto mark = [&](int k) {
    if (a.prof) {
      const long long t = clock64();
      ph[k] += static_cast<unsigned long long>(t - tmark);
      tmark = t;
    }
  };
  for (;; ++tphase) {
    mark(5);
    if (tid == 0) s_tile = atomicAdd(a.counter, 1);
    __syncthreads();
    const int qi = s_tile;
    if (qi >= a.ntiles) break;
    if (tid < 3) {
      const unsigned long long pk = a.ocoord[qi];
      const int tm = static_cast<int>((pk >> (10 * tid)) & 1023);
      const TileMode& src = a.tmode[tid][tm];
      g.tco[tid] = tm;
      g.start[tid] = src.start;
      g.ext[tid] = src.ext;
      g.nc[tid] = src.nc;
      for (int k = 0; k < 16; ++k) {
        g.cs[tid][k] = src.cs[k];
        g.cz[tid][k] = src.cz[k];
      }
      const int p = a.ntiles_mode[tid];
      g.nlo[tid] = tm + 1 < p ? a.bnd[tid][tm + 1] : a.dims[tid];
      g.flo[tid] = tm + 2 < p ? a.bnd[tid][tm + 2] : a.dims[tid];
      if (tid == 0) g.lt = a.order[qi];
    }
    __syncthreads();
    if (tid == 0) {
      g.gbase = static_cast<int64_t>(g.start[0]) + static_cast<int64_t>(g.start[1]) * a.stride[1] +
                static_cast<int64_t>(g.start[2]) * a.stride[2];
      int nch = 0;
      for (int m = 0; m < 3; ++m) {
        nch += a.dims[m] > g.flo[m] ? (a.dims[m] - g.flo[m] + E - 1) / E : 0;
        nch += g.flo[m] > g.nlo[m] ? (g.flo[m] - g.nlo[m] + E - 1) / E : 0;
      }
      g.nch = (a.dbg & 4) ? 0 : nch;
    }
    __syncthreads();
    const int nch = g.nch;

    if (warp == CW) {
      // ---------------- producer: B~ tile, eigenvector bases, update boxes ----
      if ((tid & 31) == 0) {
        if (!(a.dbg & 32768)) {
          mbar_expect_tx(&bar_x, BOX_BYTES);
          tma_load_3d(xr, &tmx, g.start[0] & ~1, g.start[1], g.start[2], &bar_x);
        }
        if (!(a.dbg & 16384)) {
          mbar_expect_tx(&bar_v, 3 * VHS * 8);
          for (int m = 0; m < 3; ++m)
            bulk_g2s(vh + m * VHS, a.vhat[m] + static_cast<int64_t>(g.tco[m]) * VHS, VHS * 8, &bar_v);
        }
        for (int c = 0; c < nch; ++c, ++gch) {
          const Chunk ch = chunk_of(g, a.dims, c);
          const int m = ch.m % 3;
          if (ch.first) {  // far: tile t+2 along m; near: tile t+1
            mark(7);
            wait_tile(a, g.lt + (ch.m < 3 ? 2 : 1) * mul[m]);
            fence_proxy_async();
            mark(6);
          }
          const int s = gch % NST;
          if (gch >= NST) mbar_wait(empty + s, ((gch / NST) - 1) & 1);
          int cc[3] = {g.start[0], g.start[1], g.start[2]};
          cc[m] = ch.k;
          mbar_expect_tx(full + s, BOX_BYTES);
          tma_load_3d(s < NSR ? ring + s * TD : xi, &tmx, cc[0] & ~1, cc[1], cc[2], full + s);
        }
      } else {
        gch += nch;
      }
      gch = __shfl_sync(0xffffffffu, gch, 0);
    } else {
      // ---------------- consumers --------------------------------------------
      double acc[3][2][4][2];
#pragma unroll
      for (int m = 0; m < 3; ++m)
#pragma unroll
        for (int rb = 0; rb < 2; ++rb)
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) acc[m][rb][cb][0] = acc[m][rb][cb][1] = 0.0;
      mark(0);
      double af[4][2], an[4][2];
      Chunk ch = chunk_of(g, a.dims, 0);
      if (nch > 0) chunk_afrag(a, g, ch.m % 3, ch.k, ch.kh, af);
      for (int c = 0; c < nch; ++c, ++gch) {
        const Chunk cn = chunk_of(g, a.dims, c + 1);
        if (c + 1 < nch) chunk_afrag(a, g, cn.m % 3, cn.k, cn.kh, an);  // next chunk's A, in flight
        const int s = gch % NST;
        mbar_wait(full + s, (gch / NST) & 1);
        if (c == 0) mark(1);
        const int m = ch.m % 3;
        const double* box = (s < NSR ? ring + s * TD : xi) + ((m == 0 ? ch.k : g.start[0]) & 1);
        if (m == 0) chunk_dmma<0>(box, af, acc[0]);
        else if (m == 1) chunk_dmma<1>(box, af, acc[1]);
        else chunk_dmma<2>(box, af, acc[2]);
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(empty + s);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) af[ks][0] = an[ks][0], af[ks][1] = an[ks][1];
        ch = cn;
      }
      mark(2);
      if (!(a.dbg & 32768)) mbar_wait(&bar_x, tphase & 1);  // B~ tile landed
      double* xo = xr + (g.start[0] & 1);  // the B~ box starts at an even row
      flush16<0>(xo, acc[0]);
      consumers_sync();
      flush16<1>(xo, acc[1]);
      consumers_sync();
      flush16<2>(xo, acc[2]);
      consumers_sync();
      // ---- diagonalised base case (ring = complex work tile) ----
      mark(3);
      if (!(a.dbg & 16384)) mbar_wait(&bar_v, tphase & 1);
      if (a.dbg & 2048) goto scatter16;
      {
      // ---- real block-diagonalised base case (ring = work tile) ----
      double* y = ring;
      const int* ex = g.ext;
      constexpr int VRI = 0, VRR = EE;
      cmode16<0, false, false, false>(xo, nullptr, y, nullptr, vh + VRI, vh + VRI, vh, ex, a.tiny);
      consumers_sync();
      cmode16<1, false, false, false>(y, nullptr, xr, nullptr, vh + VHS + VRI, vh + VHS + VRI, vh, ex, a.tiny);
      consumers_sync();
      cmode16<2, false, false, false>(xr, nullptr, y, nullptr, vh + 2 * VHS + VRI, vh + 2 * VHS + VRI, vh, ex,
                                      a.tiny);
      consumers_sync();
      const bool sing = cell_solve16(y, g, vh, a.tiny);
      consumers_sync();
      cmode16<0, false, false, false>(y, nullptr, xr, nullptr, vh + VRR, vh + VRR, vh, ex, a.tiny);
      consumers_sync();
      cmode16<1, false, false, false>(xr, nullptr, y, nullptr, vh + VHS + VRR, vh + VHS + VRR, vh, ex, a.tiny);
      consumers_sync();
      cmode16<2, false, false, false>(y, nullptr, xr, nullptr, vh + 2 * VHS + VRR, vh + 2 * VHS + VRR, vh, ex,
                                      a.tiny);
      if (sing) atomicMin(a.status, static_cast<int>(g.lt < 0x7f7f7f7e ? g.lt : 0x7f7f7f7e));
      consumers_sync();
      }
    scatter16:
      mark(4);
      // ---- scatter X_t, release ----
      const int e0 = g.ext[0], e1 = g.ext[1], e2 = g.ext[2];
      for (int l = tid; l < TT; l += CW * 32) {
        const int i0 = l & (E - 1), i1 = (l >> 4) & (E - 1), i2 = l >> 8;
        if (i0 < e0 && i1 < e1 && i2 < e2)
          a.X[g.gbase + i0 + i1 * a.stride[1] + i2 * a.stride[2]] = xr[i0 + S1 * i1 + S2 * i2];
      }
      consumers_sync();
      if (tid == 0) {
        __threadfence();
        st_release(a.flags + g.lt, a.epoch);
        if (a.trace) {
          unsigned long long tt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
          a.trace[g.lt] = tt;
        }
      }
    }
  }
  if (a.prof && (tid == 0 || tid == CW * 32)) {
    for (int k = 0; k < 8; ++k) atomicAdd(a.prof + k, ph[k]);
    if (tid == 0) atomicAdd(a.prof + 8, static_cast<unsigned long long>(tphase));
  }
}

// ---------------------------------------------------------------------------
// Decoupled variant: the producer warp runs one tile ahead of the consumers.
// It claims the next tile, publishes its geometry through a two-slot queue
// (mbarriers), loads its bases into the other half of a double-buffered
// table region and streams its first update boxes while the consumers are
// still in the previous tile's base case and scatter; the B~ tile goes into
// xr once the consumers signal that the previous tile has been scattered.
// The base case works in place in xr (each warp reads and writes only its
// own cross-section columns of a mode product), which frees the former work
// tile for a third ring stage (the ring is never touched by the consumers
// outside the update phase).  The producer also builds the tile's chunk list
// once (G16::ck: far tiles >= t+3 of every mode top down, then the t+2 rows,
// then the near groups), checks the far tiles' flags in one batched poll and
// waits per chunk only on tiles not yet released; with the forward gate
// (trailing cube, SolveArgs::gflags) it first acquires the last forward
// GEMM's tiles under the tile's right-hand side.
// ---------------------------------------------------------------------------
#ifndef L16_DNS
#define L16_DNS 3
#endif
constexpr int DNS = L16_DNS;  // ring stages of the decoupled kernel
// xr (the tile, base case in place), double-buffered bases, the ring
constexpr int D_OFF_VH = TD, D_OFF_RING = D_OFF_VH + 6 * VHS;
constexpr int D_BYTES = (D_OFF_RING + DNS * TD) * 8;
static_assert((D_OFF_RING * 8) % 128 == 0, "TMA destinations 128-byte aligned");

TSG_DEVINL void fill_geometry(const SolveArgs& a, G16& g, int q, int lane) {
  if (lane < 3) {
    const unsigned long long pk = a.ocoord[q];
    const int tm = static_cast<int>((pk >> (10 * lane)) & 1023);
    const TileMode& src = a.tmode[lane][tm];
    g.tco[lane] = tm;
    g.start[lane] = src.start;
    g.ext[lane] = src.ext;
    g.nc[lane] = src.nc;
    for (int k = 0; k < 16; ++k) {
      g.cs[lane][k] = src.cs[k];
      g.cz[lane][k] = src.cz[k];
    }
    const int p = a.ntiles_mode[lane];
    g.nlo[lane] = tm + 1 < p ? a.bnd[lane][tm + 1] : a.dims[lane];
    g.flo[lane] = tm + 2 < p ? a.bnd[lane][tm + 2] : a.dims[lane];
  }
  __syncwarp();
  if (lane == 0) {
    g.lt = a.order[q];
    g.gbase = static_cast<int64_t>(g.start[0]) + static_cast<int64_t>(g.start[1]) * a.stride[1] +
              static_cast<int64_t>(g.start[2]) * a.stride[2];
    int nch = 0;
    for (int m = 0; m < 3; ++m) {
      nch += a.dims[m] > g.flo[m] ? (a.dims[m] - g.flo[m] + E - 1) / E : 0;
      nch += g.flo[m] > g.nlo[m] ? (g.flo[m] - g.nlo[m] + E - 1) / E : 0;
    }
    g.nch = (a.dbg & 4) ? 0 : nch;
  }
  __syncwarp();
#if L16_ORDER_AB
  // far chunks of tiles >= t+3 (top down, mode after mode), then the lowest
  // far chunk of every mode (tile t+2's rows, released last), then near
  if (lane == 0) {
    int n[3], c = 0;
    for (int m = 0; m < 3; ++m) n[m] = a.dims[m] > g.flo[m] ? (a.dims[m] - g.flo[m] + E - 1) / E : 0;
    for (int m = 0; m < 3; ++m)
      for (int j = n[m] - 1; j >= 1; --j) {
        const int k = g.flo[m] + E * j;
        g.ck[c++] = pack_chunk(Chunk{m, k, min(k + E, a.dims[m]), 0});
      }
    for (int m = 0; m < 3; ++m)
      if (n[m] > 0) g.ck[c++] = pack_chunk(Chunk{m, g.flo[m], min(g.flo[m] + E, a.dims[m]), 0});
    for (int m = 0; m < 3; ++m) {
      const int lo = g.nlo[m], hi = g.flo[m];
      const int nn = hi > lo ? (hi - lo + E - 1) / E : 0;
      for (int j = 0; j < nn; ++j) g.ck[c++] = pack_chunk(Chunk{m + 3, lo + E * j, hi, j == 0});
    }
  }
#else
  for (int c = lane; c < g.nch; c += 32) g.ck[c] = pack_chunk(chunk_of(g, a.dims, c));
#endif
  __syncwarp();
}

__global__ void __launch_bounds__(THREADS, 1)
    solve_lap16d_kernel(SolveArgs a, const __grid_constant__ CUtensorMap tmx) {
  // with the forward gate, right-hand sides are awaited per tile instead
  if (!a.gflags) pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) double smem[];
  __shared__ G16 gq[2];
  __shared__ __align__(8) uint64_t full[DNS], empty[DNS], bar_x, bar_v[2], info_full[2], info_empty[2], xr_free;
  double* xr = smem;
  double* vhb = smem + D_OFF_VH;
  double* ring = smem + D_OFF_RING;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < DNS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, CW);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_v + s, 1);
      mbar_init(info_full + s, 1);
      mbar_init(info_empty + s, 1);
    }
    mbar_init(&bar_x, 1);
    mbar_init(&xr_free, 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t mul[3] = {1, a.ntiles_mode[0], static_cast<int64_t>(a.ntiles_mode[0]) * a.ntiles_mode[1]};

  if (warp == CW) {
    // ---------------- producer warp ----------------
    unsigned gch = 0;
    for (int it = 0;; ++it) {
      const int slot = it & 1;
      if (it >= 2) mbar_wait(&info_empty[slot], ((it >> 1) - 1) & 1);
      G16& g = gq[slot];
      int q = 0;
      if (lane == 0) q = atomicAdd(a.counter, 1);
      q = __shfl_sync(0xffffffffu, q, 0);
      const bool done = q >= a.ntiles;
      if (!done) fill_geometry(a, g, q, lane);
      if (lane == 0) g.done = done ? 1 : 0;
#if L16_TRACE2
      if (lane == 0 && !done && a.trace) {
        unsigned long long tt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
        a.trace[a.ntiles_total + g.lt] = tt;  // claimed
      }
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(&info_full[slot]);
      if (done) break;
      if (a.gflags) {
        // forward gate: the GEMM tiles holding this tile's right-hand side
        // (rows i0 + n0 i1 for i1 in the tile, one lane per i1)
        if (lane < g.ext[1]) {
          const int r0 = g.start[0] + a.dims[0] * (g.start[1] + lane);
          const int mlo = r0 / a.gbm, mhi = (r0 + g.ext[0] - 1) / a.gbm;
          const int nlo = g.start[2] / a.gbn, nhi = (g.start[2] + g.ext[2] - 1) / a.gbn;
          for (int nt = nlo; nt <= nhi; ++nt)
            for (int mt = mlo; mt <= mhi; ++mt) {
              const int* f = a.gflags + mt + nt * a.gtm;
              // bounded: the gating GEMM must run beside this grid; if it
              // cannot (serialised launches), fail the solve instead of hanging
              long long spins = 0;
              while (ld_acquire(f) != a.gepoch) {
                __nanosleep(64);
                if (++spins > ((a.dbg & 32768) ? 2000000LL : (1LL << 26))) {
                  atomicMin(a.status, kGateTimeout);
                  break;
                }
              }
            }
        }
        __syncwarp();
        fence_proxy_async();
      }
      if (lane == 0) {  // the tile's bases first (no dependency)
        double* vh = vhb + slot * 3 * VHS;
        mbar_expect_tx(&bar_v[slot], 3 * VHS * 8);
        for (int m = 0; m < 3; ++m)
          bulk_g2s(vh + m * VHS, a.vhat[m] + static_cast<int64_t>(g.tco[m]) * VHS, VHS * 8, &bar_v[slot]);
      }
      // far groups: which tiles above t+1 are already released?  lanes
      // 10 m + j read the flag of tile t + (2 + j) e_m; released tiles along
      // a mode form a suffix, so the lowest offset with every offset above
      // it released confirms all those tiles (rdy[m]: lowest confirmed tile
      // index along m; ten released offsets confirm everything from t+2 up)
      int rdy[3];
      {
        const int pm = lane / 10, off = 2 + lane % 10;
        bool okf = true;
        if (pm < 3 && g.tco[pm] + off < a.ntiles_mode[pm])
          okf = ld_acquire(a.flags + g.lt + off * mul[pm]) >= a.epoch;
        const unsigned bal = __ballot_sync(0xffffffffu, okf);
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          const unsigned bits = (bal >> (10 * m)) & 0x3ffu;  // bit j: offset 2 + j
          int o = 12;                                      // lowest offset of the released suffix
          while (o > 2 && ((bits >> (o - 3)) & 1u)) --o;
          rdy[m] = o == 12 ? a.ntiles_mode[m] : g.tco[m] + o;
          if (bits == 0x3ffu) rdy[m] = g.tco[m] + 2;
        }
        __syncwarp();
        fence_proxy_async();
      }
      if (lane == 0) {
        const int nch = g.nch;
        bool bx = false;
        auto issue_bx = [&]() {
          if (it >= 1) mbar_wait(&xr_free, (it - 1) & 1);  // previous tile scattered
          mbar_expect_tx(&bar_x, BOX_BYTES);
          tma_load_3d(xr, &tmx, g.start[0] & ~1, g.start[1], g.start[2], &bar_x);
          bx = true;
        };
        // B~ box: at once when the previous tile is already scattered (ramp
        // regimes: the consumers idle), else after the ring is filled
        if (nch == 0 || it == 0 || mbar_test(&xr_free, (it - 1) & 1)) issue_bx();
        for (int c = 0; c < nch; ++c, ++gch) {
          const Chunk ch = unpack_chunk(g.ck[c]);
          const int m = ch.m % 3;
          if (ch.m < 3) {  // far chunk: the tile holding its first row
            const int tk = a.rowtile[m][ch.k];
            if (tk < rdy[m]) {
              wait_tile(a, g.lt + (tk - g.tco[m]) * mul[m]);
              fence_proxy_async();
              rdy[m] = tk;
            }
          } else if (ch.first) {
            wait_tile(a, g.lt + mul[m]);
            fence_proxy_async();
          }
          const int s = gch % DNS;
          if (gch >= DNS) mbar_wait(empty + s, ((gch / DNS) - 1) & 1);
          // box origin: the chunk's first row along m, the tile's start elsewhere
          const int c0 = m == 0 ? ch.k : g.start[0], c1 = m == 1 ? ch.k : g.start[1],
                    c2 = m == 2 ? ch.k : g.start[2];
          mbar_expect_tx(full + s, BOX_BYTES);
          tma_load_3d(ring + s * TD, &tmx, c0 & ~1, c1, c2, full + s);
          if (!bx && (c == DNS - 1 || c + 1 == nch)) issue_bx();  // ring filled first
        }
      }
      __syncwarp();
    }
  } else {
    // ---------------- consumers ----------------
    unsigned gch = 0;
    // -DL16_PROF=1 + TSG_PROF: consumer thread 0 accumulates cycles per
    // phase (compiled out by default: the counters cost registers)
#if L16_PROF
    const bool prof = a.prof != nullptr && tid == 0;
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tm0 = clock64();
    auto mark = [&](int k) {
      if (prof) {
        const long long t = clock64();
        ph[k] += static_cast<unsigned long long>(t - tm0);
        tm0 = t;
      }
    };
    int ntl = 0;
#else
    auto mark = [](int) {};
#endif
    for (int it = 0;; ++it) {
      const int slot = it & 1;
      mbar_wait(&info_full[slot], (it >> 1) & 1);
      const G16& g = gq[slot];
      mark(0);
      if (g.done) break;
#if L16_PROF
      ++ntl;
#endif
      const int nch = g.nch;
      double acc[3][2][4][2];
#pragma unroll
      for (int m = 0; m < 3; ++m)
#pragma unroll
        for (int rb = 0; rb < 2; ++rb)
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) acc[m][rb][cb][0] = acc[m][rb][cb][1] = 0.0;
      double af[4][2], an[4][2];
      Chunk ch = nch > 0 ? unpack_chunk(g.ck[0]) : Chunk{0, 0, 0, 0};
      if (nch > 0) chunk_afrag(a, g, ch.m % 3, ch.k, ch.kh, af);
      for (int c = 0; c < nch; ++c, ++gch) {
        const Chunk cn = c + 1 < nch ? unpack_chunk(g.ck[c + 1]) : Chunk{0, 0, 0, 0};
        if (c + 1 < nch) chunk_afrag(a, g, cn.m % 3, cn.k, cn.kh, an);
        const int s = gch % DNS;
#if L16_TRACE2
        if (tid == 0 && a.trace && ch.m >= 3 && (c == 0 || unpack_chunk(g.ck[c - 1]).m < 3)) {
          unsigned long long tt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
          a.trace[2 * a.ntiles_total + g.lt] = tt;  // far groups done
        }
#endif
        mbar_wait(full + s, (gch / DNS) & 1);
        const int m = ch.m % 3;
        const double* box = ring + s * TD + ((m == 0 ? ch.k : g.start[0]) & 1);
        if (m == 0) chunk_dmma<0>(box, af, acc[0]);
        else if (m == 1) chunk_dmma<1>(box, af, acc[1]);
        else chunk_dmma<2>(box, af, acc[2]);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) af[ks][0] = an[ks][0], af[ks][1] = an[ks][1];
        ch = cn;
      }
      mark(1);
#if L16_TRACE2
      if (tid == 0 && a.trace) {
        unsigned long long tt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
        a.trace[3 * a.ntiles_total + g.lt] = tt;  // all chunks done
      }
#endif
      mbar_wait(&bar_x, it & 1);
      mark(2);
      double* xo = xr + (g.start[0] & 1);
      // Warp w owns the cross-section columns [32 w, 32 w + 32) of every
      // mode; for modes 0 and 1 these are the whole slab i2 in {2w, 2w+1},
      // so mode-0 and mode-1 passes of the same warp need no CTA barrier
      // between them (mode 2, the cell solve and the scatter do).
      flush16<2>(xo, acc[2]);
      consumers_sync();
      flush16<0>(xo, acc[0]);
      __syncwarp();
      flush16<1>(xo, acc[1]);
      mark(3);
      mbar_wait(&bar_v[slot], (it >> 1) & 1);
      mark(4);
      const double* vh = vhb + slot * 3 * VHS;
      const int* ex = g.ext;
      constexpr int VRI = 0, VRR = EE;
      __syncwarp();
      cmode16<0, false, false, false>(xo, nullptr, xo, nullptr, vh + VRI, vh + VRI, vh, ex, a.tiny);
      __syncwarp();
      cmode16<1, false, false, false>(xo, nullptr, xo, nullptr, vh + VHS + VRI, vh + VHS + VRI, vh, ex, a.tiny);
      consumers_sync();
      cmode16<2, false, false, false>(xo, nullptr, xo, nullptr, vh + 2 * VHS + VRI, vh + 2 * VHS + VRI, vh, ex,
                                      a.tiny);
      consumers_sync();
      const bool sing = cell_solve16(xo, g, vh, a.tiny);
      consumers_sync();
      // back to the Schur basis: mode 2 first, then the warp-local modes 0, 1
      cmode16<2, false, false, false>(xo, nullptr, xo, nullptr, vh + 2 * VHS + VRR, vh + 2 * VHS + VRR, vh, ex,
                                      a.tiny);
      consumers_sync();
      cmode16<0, false, false, false>(xo, nullptr, xo, nullptr, vh + VRR, vh + VRR, vh, ex, a.tiny);
      __syncwarp();
      cmode16<1, false, false, false>(xo, nullptr, xo, nullptr, vh + VHS + VRR, vh + VHS + VRR, vh, ex, a.tiny);
      if (sing) atomicMin(a.status, static_cast<int>(g.lt < 0x7f7f7f7e ? g.lt : 0x7f7f7f7e));
      consumers_sync();
      mark(5);
      const int e0 = g.ext[0], e1 = g.ext[1], e2 = g.ext[2];
      for (int l = tid; l < TT; l += CW * 32) {
        const int i0 = l & (E - 1), i1 = (l >> 4) & (E - 1), i2 = l >> 8;
        if (i0 < e0 && i1 < e1 && i2 < e2)
          a.X[g.gbase + i0 + i1 * a.stride[1] + i2 * a.stride[2]] = xo[i0 + S1 * i1 + S2 * i2];
      }
      fence_proxy_async();  // this thread's generic xr / xi accesses before the next TMA into them
      consumers_sync();
      if (tid == 0) {
        __threadfence();
        st_release(a.flags + g.lt, a.epoch);
        if (a.trace) {
          unsigned long long tt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
          a.trace[g.lt] = tt;
        }
        mbar_arrive(&xr_free);
        mbar_arrive(&info_empty[slot]);
      }
      mark(6);
    }
#if L16_PROF
    if (prof) {
      for (int k = 0; k < 7; ++k) atomicAdd(a.prof + k, ph[k]);
      atomicAdd(a.prof + 8, static_cast<unsigned long long>(ntl));
    }
#endif
  }
}

}  // namespace

TileCaps solve_lap16_caps() { return TileCaps{E, TT, EE}; }

#ifndef L16_DEC
#define L16_DEC 1
#endif
bool lap16_decoupled() { return L16_DEC || std::getenv("TSG_L16DEC"); }

cudaError_t launch_solve_lap16(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info) {
  if (a.ntiles <= 0) return cudaSuccess;
  CUtensorMap map;
  const uint64_t dims[3] = {static_cast<uint64_t>(a.dims[0]), static_cast<uint64_t>(a.dims[1]),
                            static_cast<uint64_t>(a.dims[2])};
  const uint32_t box[3] = {BX, BY, BZ};
  if (!encode_tmap_f64(&map, a.X, 3, dims, box)) return cudaErrorInvalidValue;
  if (lap16_decoupled()) {
    int nsm2 = 0, occ2 = 0;
    if (cudaError_t e = kernel_setup(solve_lap16d_kernel, D_BYTES, THREADS, &nsm2, &occ2); e != cudaSuccess)
      return e;
    int64_t grid = nsm2;
    if (grid > a.ntiles) grid = a.ntiles;
    if (a.max_grid > 0 && grid > a.max_grid) grid = a.max_grid;
    if (info) *info = SolveLaunchInfo{static_cast<int>(grid), THREADS, D_BYTES, 1};
    if (a.gflags && !a.gate_pdl) {  // gated on the NEXT kernel's output: plain launch
      solve_lap16d_kernel<<<static_cast<unsigned>(grid), THREADS, D_BYTES, st>>>(a, map);
      return cudaGetLastError();
    }
    cudaError_t le = launch_pdl(solve_lap16d_kernel, static_cast<unsigned>(grid), THREADS, D_BYTES, st, a, map);
    return le != cudaSuccess ? le : cudaGetLastError();
  }
  int nsm = 0, occ = 0;
  if (cudaError_t e = kernel_setup(solve_lap16_kernel, BYTES, THREADS, &nsm, &occ); e != cudaSuccess) return e;
  int64_t grid = nsm;
  if (grid > a.ntiles) grid = a.ntiles;
  if (info) *info = SolveLaunchInfo{static_cast<int>(grid), THREADS, BYTES, 1};
  cudaError_t le = launch_pdl(solve_lap16_kernel, static_cast<unsigned>(grid), THREADS, BYTES, st, a, map);
  return le != cudaSuccess ? le : cudaGetLastError();
}

}  // namespace tsg
