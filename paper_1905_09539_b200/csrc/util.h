#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tsg {
// *out_dev += sum_i x_i^2  (out_dev must be zeroed by the caller)
cudaError_t sumsq(const double* x, int64_t n, double* out_dev, cudaStream_t st);
// y += a * x
cudaError_t axpy(double* y, const double* x, double a, int64_t n, cudaStream_t st);
// Per-solve state reset in one launch: flags[0..nf) = 0, counter[0] = 0,
// counter[1] = status (no singular cell), extra[0..ne) = 0 (may be null).
cudaError_t reset_state(int* flags, int64_t nf, int* counter, int status, int* extra, int64_t ne,
                        cudaStream_t st);
}  // namespace tsg
