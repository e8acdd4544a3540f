// Host-side interface of the DMMA batched GEMM (gemm.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tsg {

// C[b] = alpha * A[b] * B[b] + beta * C[b], column-major, b in [0, batch):
//   A[b](m,k) = A[b*sA + m + k*lda],  B[b](k,n) = B[b*sB + k + n*ldb],
//   C[b](m,n) = C[b*sC + m + n*ldc].
struct GemmArgs {
  const double* A;
  const double* B;
  double* C;
  int M, N, K;
  int64_t lda, ldb, ldc;
  int64_t sA, sB, sC;
  int64_t batch;
  double alpha, beta;
  // Optional tile-flag gate (back transform overlapped with the solve): the
  // CTA owning columns [n0, n0+BN) of a mode-0 product first waits until
  // wflags[wids[i]] == wepoch for i in [woff[n0/64], woff[ceil((n0+BN)/64)]);
  // n-tiles are then issued last-column first, and with pdl the kernel is
  // launched as a programmatic dependent of the preceding solve kernel.
  const int* wflags = nullptr;
  const int* woff = nullptr;
  const int* wids = nullptr;
  int wepoch = 0;
  int wgroups = 0;  // number of 64-column groups (entries of woff minus one)
  int pdl = 0;
  // Producer side of a slab-wise chain (mode-0 product feeding mode 1,
  // batch 1): each CTA releases dflags[mt + nt * tiles_m] = depoch after
  // its stores.
  int* dflags = nullptr;
  int depoch = 0;
  // Consumer side (batched mode-1 product): batch q reads producer columns
  // [q * pcpb, (q + 1) * pcpb), i.e. producer tiles (all ptm m-tiles) x
  // (n-tiles of width pbn over those columns); the CTA acquires their flags
  // (== pepoch) instead of waiting for the whole producer grid.  pdesc:
  // batches are issued last first (the producer finishes those first).
  const int* pflags = nullptr;
  int pepoch = 0, ptm = 0, pbn = 0, pcpb = 0, pdesc = 0;
  // nowait: a programmatic launch whose inputs are complete by construction
  // (skip griddepcontrol.wait); drev: issue the CTA tiles last first.
  int nowait = 0, drev = 0;
};

// CTA tile (BM x BN) dgemm_nn uses for an M x N product (0 x 0: unknown).
void gemm_tile_shape(int M, int N, int* bm, int* bn);

// Column granularity of the GemmArgs tile-flag gate.
constexpr int kWaitCols = 64;

cudaError_t dgemm_nn(const GemmArgs& g, cudaStream_t st);
// Set the launch attributes of every GEMM kernel (idempotent; plans call it
// at creation so no attribute change lands inside a launch chain).
cudaError_t gemm_prepare();

// TMA-staged variant (gemm_tma.cu): the same product with the operand tiles
// moved by cp.async.bulk.tensor into swizzled stages behind mbarriers.
// gemm_tma_ok: the call has no tile-flag gates and its operands satisfy the
// tensor-map alignment rules (16-byte base and strides).
bool gemm_tma_ok(const GemmArgs& g);
cudaError_t dgemm_nn_tma(const GemmArgs& g, cudaStream_t st);
cudaError_t gemm_tma_prepare();

// Y = X x_mode A for a dense tensor (tensor.hpp:187-231 semantics):
// A is r x dims[mode] column-major (device), At = A^T (n x r, device; only
// used for mode > 0).  Y has dims[mode] replaced by r.
cudaError_t mode_product(const double* X, double* Y, int d, const int* dims, int mode,
                         const double* A, const double* At, int r, double alpha, double beta,
                         cudaStream_t st, double* flops = nullptr,
                         const GemmArgs* gate = nullptr);

// Fused small-mode transform (modes_small.cu): Y = X x_a A (x_{a+1} B when
// pair), one HBM pass; extents 16, 24, 32, 40 only (small_mode_ok).
bool small_mode_ok(int n);
// The fused pass over mode a (and a + 1 when pair) is available for this
// shape (extents as above and whole 8-fibre blocks per shared-memory block).
bool small_pass_ok(int d, const int* dims, int a, bool pair);
cudaError_t mode_pair_small(const double* X, double* Y, int d, const int* dims, int a, bool pair,
                            const double* A, const double* B, cudaStream_t st, double* flops = nullptr);

}  // namespace tsg
