// Host-side interface of the reduced-form dataflow solver (solve.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tsg {

constexpr int kMaxOrder = 8;
constexpr int kEigStride = 12;  // doubles of normal-form data per Schur-block start row
constexpr int kPStride = 20;    // doubles of eigenbasis (P, Pinv, lambda) data per block row

constexpr int kMaxCells = 32;   // Schur cells per mode inside one tile
constexpr int kMaxSlabs = 8;    // slabs (ranks) along the last mode, sharded solves

// Host-built geometry of tile index t along one mode: global start, extent,
// and its 1x1/2x2 Schur cells (start offset inside the tile, size).
struct alignas(16) TileMode {
  int start;
  unsigned char ext, nc, pair, pad;
  unsigned char cs[kMaxCells], cz[kMaxCells];
  unsigned char cellof[kMaxCells];  // tile row -> cell index
  unsigned char cend[kMaxCells];    // tile row -> first row after its cell
  unsigned char cplx[kMaxCells];    // 1 on the first row of a 2x2 block
  unsigned char ckind[kMaxCells];   // 1/2: first/second row of a complex-eigenvalue pair, else 0
  float vcond;                      // lap3: ||V||_F ||V^-1||_F / ext of the block's eigenvectors
  int far_lo;                       // first row of tile t+3 (the mode extent when there is none)
};

// lap3 diagonalised tiles: per tile index along a mode, V^{-1} (re, im),
// V (re, im) as 8x8 row-major (identity-padded) and lambda (re, im).
constexpr int kVhStride = 4 * 64 + 2 * 8;
constexpr int kVhStride16 = 2 * 256 + 2 * 16;  // real block-diagonal basis (lap16)
// A tile is diagonalised when the product of its three vcond values is at
// most this (the eigenvector transforms then cost <= ~kDiagCond ulps).
constexpr float kDiagCond = 1000.0f;

// Reduced Laplace-like / gsylv equation on a tiled tensor, solved in place
// by one persistent dataflow kernel (see solve.cu for the algorithm).
struct SolveArgs {
  int family;                   // 0 Laplace, 1 gsylv
  int d;
  int dims[kMaxOrder];
  int64_t stride[kMaxOrder];    // element strides (mode 0 fastest)
  double* X;                    // B~ on entry, X~ on exit (device)
  // gsylv auxiliaries (family 1): chain partial products W_m of solved
  // tiles, W[d-1] = X x_{d-1} A_{d-1}, W[m] = W[m+1] x_m A_m, W[1] = V.
  double* W[kMaxOrder];
  const double* T[kMaxOrder];   // quasi-triangular coefficients (device, col-major)
  const double* Tc;             // gsylv: upper-triangular C factor (mode 0)
  const TileMode* tmode[kMaxOrder];  // per mode: ntiles_mode entries
  const double* eig[kMaxOrder]; // per row: kEigStride doubles (valid at block starts)
  int ntiles_mode[kMaxOrder];
  const int* bnd[kMaxOrder];    // tile boundaries per mode (ntiles_mode+1)
  const int* rowtile[kMaxOrder];  // per mode: tile index of every row
  int64_t ntiles;
  const int* order;             // topological order of linear tile ids
  const unsigned long long* ocoord;  // packed tile coordinates of order[] (10 bits/mode)
  const double* pdat[kMaxOrder];     // per row: kPStride doubles (fast Laplace path)
  const double* dhat[kMaxOrder];     // per tile index: eigenbasis diag block + lambdas (lap3)
  const double* vhat[kMaxOrder];     // per tile index: eigenvectors of the diag block (lap3)
  int* flags;                   // per tile: epoch when solved
  int* counter;                 // work queue head (zeroed before launch)
  int* status;                  // first singular cell linear index (or INT_MAX)
  int epoch;
  double tiny;                  // |cell eigenvalue| <= tiny -> singular
  int refine;                   // 1: one refinement step per base cell
  int dbg;                      // ablation mask (development only; 0 in production)
  unsigned long long* prof;     // optional per-phase cycle counters (development)
  unsigned long long* trace;    // optional per-tile release globaltimer (development)
  // Slabs along the last mode (lap3 only; nslab = 1 and xs[0] = X otherwise).
  // Element offset(i) of the global tensor lives at xs[q] + offset(i) for
  // the slab q = slab_of(i_{d-1}); xs[q] are virtual bases (slab pointer
  // minus slo[q] * stride[d-1]), peer-mapped on multi-GPU runs.
  int tlog[kMaxOrder];          // solve_lapd: log2 padded tile extent per mode
  int tsh[kMaxOrder];           // solve_lapd: bit offset of mode m in the tile index
  int nslab;
  int sys;                      // 1: flags and tiles shared across GPUs (system scope)
  int slo[kMaxSlabs + 1];       // slab row bounds along mode d-1 (tile-aligned)
  double* xs[kMaxSlabs];
  int* fs[kMaxSlabs];           // tile flags of the slab owner (indexed by linear tile id)
  // Forward gate (lap16d): the last forward GEMM (mode 2: rows i0 + n0 i1,
  // columns i2) releases each gbm x gbn output tile as gflags[mt + nt * gtm]
  // = gepoch; a tile loads its right-hand side once the GEMM tiles covering
  // it are released (null: the whole forward pass precedes the launch).
  const int* gflags;
  int gepoch, gbm, gbn, gtm;
  int max_grid;                 // > 0: at most this many CTAs (lap16d)
  int gate_pdl;                 // with gflags: launch as a programmatic dependent of the gating GEMM
  int64_t ntiles_total;         // all tiles of the plan (trace layout; development)
};

// SolveArgs::status value of a forward gate that never opened (lap16d).
constexpr int kGateTimeout = -2;  // negative: atomicMin keeps it over any tile index

struct SolveLaunchInfo {
  int grid, block, smem_bytes, ctas_per_sm;
};

// Per-order tile caps the host tiler must honour (e_m <= emax, prod <= Emax,
// prod/e_m <= nmax).
struct TileCaps {
  int emax, Emax, nmax;
};
TileCaps solve_caps(int family, int d);

cudaError_t launch_solve(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info);

// Order-3 Laplace fast path (solve_lap3.cu): padded 16^3 tiles.
TileCaps solve_lap3_caps(int lt);  // lt = log2 tile extent (3 or 4)
cudaError_t launch_solve_lap3(int lt, const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info);

// Order-3 Laplace, 16^3 tiles, TMA-staged updates, diagonalised base case
// (solve_lap16.cu; plans whose tiles are all diagonalisable).
TileCaps solve_lap16_caps();
cudaError_t launch_solve_lap16(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info);
// true when launch_solve_lap16 runs the decoupled kernel (solve_lap16d_kernel)
bool lap16_decoupled();

// Higher-order Laplace (solve_lapd.cu, d = 4..6): small padded tiles,
// DMMA updates, diagonalised base case.
TileCaps solve_lapd_caps();
cudaError_t launch_solve_lapd(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info);

// gsylv d = 3..5 (solve_gsyd.cu): small tiles, DMMA chain updates, tail
// eigenbasis + mode-0 pencil back substitution.
TileCaps solve_gsyd_caps();
cudaError_t launch_solve_gsyd(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info);

// Fast Laplace path (solve_lap.cu): small tiles, eigenbasis base cells.
TileCaps solve_lap_caps(int d);
cudaError_t launch_solve_lap(const SolveArgs& a, cudaStream_t st, SolveLaunchInfo* info);

// ---- Eigen-decoupled fibre solve (solve_fibre.cu) ---------------------------
// Modes s in S are moved into their real block-eigenbasis by the transforms
// (T_s = P_s Lambda_s P_s^{-1}, Lambda_s = 1x1 lambda / 2x2 [[re, im], [-im, re]]
// blocks), so the reduced operator is
//     sum_{s in S} X x_s Lambda_s  +  X x_f T_f
// and splits into independent units (one Schur cell per S mode) of 2^k
// coupled fibres along the one free mode f (k = complex cells in the unit).
// A butterfly over the unit's complex cells turns them into 2^(k-1) complex
// fibres, each solving (T_f + sigma I) z = r by back substitution over the
// 1x1/2x2 cells of T_f.  Mode 0 is in S (f > 0) and is cut into chunks of
// whole cells; a block = one chunk x one cell of every other S mode x the
// whole f extent.
struct FibreCell {
  int start, size;
  double re, im;  // 1x1: lambda = re; 2x2: Lambda block [[re, im], [-im, re]]
};
constexpr int kFibreMaxS = 6;
// Per mode-0 cell of a chunk (host-built, chunk_u0 indexes the chunk's first):
// row offset in the chunk, 2x2 flag, pairs before it in the chunk, and its
// contribution to the shift (re, -omega for a pair).
struct alignas(16) FibreUnit {
  int rl0, pair0, npair_before, pad;
  double sr, si;
};
struct FibreArgs {
  double* X;                 // in place: B^ on entry, X^ on exit
  int nf;                    // extent of the free mode f
  int64_t sf;                // its stride
  const double* Tt;          // T_f row-major (Tt[i * nf + j] = T_f(i, j)); gsylv: S
  int gs;                    // 1: gsylv pencil fibres (S + z Tc) x = b, f = 0, z a product of eigenvalues
  const double* Tct;         // gsylv: Tc row-major
  int64_t sc;                // stride of the chunk mode (Laplace: mode 0, 1; gsylv: mode 1, n_0)
  const double* fcell;       // per row of f: 4 doubles (code 0/1/2, a, omega, unused)
  int nchunk;
  const int* chunk_lo;       // nchunk + 1 mode-0 row bounds (whole cells)
  const int* cellrow0;       // mode-0 row -> cell index
  const FibreCell* cell0;    // mode-0 cells
  const int* chunk_u0;       // nchunk + 1: first unit of every chunk
  const FibreUnit* units;    // mode-0 cells as units, chunk by chunk
  int cell_smem;             // > 0: cache the S' cell tables (this many) in shared memory
  int ns;                    // other S modes
  int64_t sstride[kFibreMaxS];
  int ncell[kFibreMaxS];
  const FibreCell* cells[kFibreMaxS];
  int64_t nblocks;
  int maxcol;                // largest block width (columns = chunk rows x 2^k')
  int small;                 // 1: the register kernel (n_f <= 24, chunks <= 128 rows)
  int big;                   // 1: the DMMA-blocked kernel (row blocks rb, shared pitch)
  int wide;                  // 1: the warp-group kernel (fibre_wide_kernel; rows blocks <= 16)
  int pitch;                 // big/wide: shared row pitch (= 4 mod 16 doubles)
  int nrb;                   // big/wide: row blocks of f (<= 8 rows, whole cells)
  const int* rb;             // big/wide: nrb + 1 row-block bounds
  const unsigned* rbcode;    // wide: per row block, 2 bits per row (0 1x1, 1/2 rows of a 2x2 cell)
  int* counter;              // block queue head (zeroed before launch)
  int* status;               // first singular element offset (atomicMin)
  double tiny;
  unsigned long long* prof;  // -DWIDE_PROF=1 builds: per-phase cycle sums (TSG_PROF)
};
cudaError_t launch_fibre_solve(const FibreArgs& a, int device, cudaStream_t st, SolveLaunchInfo* info);
bool fibre_small_ok(int nf, int chunk_w);
int fibre_pitch(int maxcol);
size_t fibre_big_smem(int nf, int maxcol, int cell_smem);
// wide kernel: columns per block (maxcol bound) and its shared memory
constexpr int kWideCols = 32;
size_t fibre_wide_smem(int nf, int maxcol, int cell_smem, int nrb = 0, int gs = 0);

}  // namespace tsg
