#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tsg {
// *out_dev += sum_i x_i^2  (out_dev must be zeroed by the caller)
cudaError_t sumsq(const double* x, int64_t n, double* out_dev, cudaStream_t st);
// y += a * x
cudaError_t axpy(double* y, const double* x, double a, int64_t n, cudaStream_t st);
// Per-solve state reset in one launch: flags[0..nf) = 0, counter[0] = 0,
// extra[0..ne) = 0 (may be null).  The status word counter[1] is sticky
// across solves: the host re-arms it when it reads it (plan.cpp).
cudaError_t reset_state(int* flags, int64_t nf, int* counter, int* extra, int64_t ne, cudaStream_t st);

// Re-sharding pack / unpack of the decoupled multi-GPU solve (dist.py): `rows`
// contiguous runs of n0 doubles <-> nranks segments, segment q holding columns
// [b0[q], b0[q+1]) of every run ((rows, w_q) row-major, at offset rows * b0[q]).
// dir 0: runs -> segments (pack), 1: segments -> runs (unpack).
constexpr int kMaxPackRanks = 64;
cudaError_t slab_pack(const double* src, double* dst, int64_t rows, int n0, int nranks, const int* b0,
                      int dir, cudaStream_t st);

// Launch setup of a kernel on the CURRENT device, thread-safe and cached per
// (kernel, device, smem, threads): raises the dynamic shared-memory opt-in
// when smem exceeds what was set before, and returns the SM count and the
// resident CTAs per SM (>= 1).  Several contexts on different devices (one
// per host thread, include/tsylv_gpu.h) each get their own attribute.
cudaError_t kernel_setup(const void* fn, size_t smem, int threads, int* nsm, int* occ);
template <typename K>
cudaError_t kernel_setup(K* fn, size_t smem, int threads, int* nsm, int* occ) {
  return kernel_setup(reinterpret_cast<const void*>(fn), smem, threads, nsm, occ);
}
}  // namespace tsg
