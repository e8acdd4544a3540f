// Complex-scalar device path (zsolve.cu): interleaved (re, im) FP64 buffers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tsg {

constexpr int kZMaxOrder = 8;

// C[b] = alpha A[b] B[b] + beta C[b] (complex, column-major; leading
// dimensions and batch strides in complex elements; alpha, beta real).
struct ZGemmArgs {
  const double* A;
  const double* B;
  double* C;
  int M, N, K;
  int64_t lda, ldb, ldc;
  int64_t sA, sB, sC;
  int64_t batch;
  double alpha, beta;
};
cudaError_t zgemm(const ZGemmArgs& g, cudaStream_t st);

// Y = X x_mode A (tensor.hpp:187-231 for T = Complex); A is r x dims[mode]
// column-major, At = A^T (plain transpose; only read for mode > 0).
cudaError_t zmode_product(const double* X, double* Y, int d, const int* dims, int mode,
                          const double* A, const double* At, int r, double alpha, double beta,
                          cudaStream_t st, double* flops = nullptr);

// Decoupled fibre solve along mode f, in place on x:
//   (S + z Tc) x_fibre = r_fibre,  z = sum_m lam_m[i_m] (product = 0,
//   Laplace; Tc = NULL means the identity) or prod_m lam_m[i_m] (product =
//   1, gsylv) over the modes m != f.  St / Tct are row-major (transposed).
// Blocked: rows of f in blocks of 32 from the bottom; the coupling to the rows
// already solved is a complex DMMA GEMM with the off-diagonal block of S (and
// of Tc against the z-scaled solved rows kept in `work`), the 32-row diagonal
// block is substituted per fibre from shared memory (zfibre_kernel).  S / Tc
// are the column-major copies (needed for f = 0), work holds N complex
// elements (gsylv only).
struct ZFibreArgs {
  double* x;
  int d, f, nf;
  int dims[kZMaxOrder];
  int64_t sf;    // stride of mode f (complex elements)
  int64_t nfib;  // N / nf
  const double* St;
  const double* Tct;
  const double* S;    // column-major S (f = 0 updates); may be null when f > 0
  const double* Tc;   // column-major Tc (gsylv)
  double* work;       // gsylv: z x of the solved rows (N complex elements)
  int i_lo, i_hi;     // rows of the diagonal block of one launch (set by zfibre_solve)
  const double* lam;  // packed eigenvalues, mode m at lam_off[m]
  int lam_off[kZMaxOrder];
  int product;
  double tiny2;  // |pivot|^2 <= tiny2 -> singular (status = min fibre index)
  int* status;
};
cudaError_t zfibre_solve(const ZFibreArgs& a, cudaStream_t st, int* launches = nullptr, double* flops = nullptr);

// Fully triangular reduced Laplace solve by wavefronts (one launch per
// level); Tt[m] row-major T_m.  x: B~ in, X~ out.
struct ZLevelArgs {
  double* x;
  int d, m0, level;
  int dims[kZMaxOrder];
  int64_t stride[kZMaxOrder];
  const double* Tt[kZMaxOrder];
  int64_t nred;  // N / dims[m0]
  double tiny2;
  int* status;
};
cudaError_t zlevel_solve(ZLevelArgs a, cudaStream_t st, int* launches = nullptr);

}  // namespace tsg
