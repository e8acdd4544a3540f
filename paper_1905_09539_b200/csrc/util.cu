// Small device utilities: squared Frobenius norms and fused r -= t, used by
// the device residual (tsg_residual; reference oracle.hpp:231-268).
#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "util.h"

namespace tsg {
namespace {

__global__ void sumsq_kernel(const double* __restrict__ x, int64_t n, double* out) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = x[i];
    s = fma(v, v, s);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double ws[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) ws[w] = s;
  __syncthreads();
  if (w == 0) {
    s = lane < (blockDim.x >> 5) ? ws[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) atomicAdd(out, s);
  }
}

__global__ void axpy_kernel(double* __restrict__ y, const double* __restrict__ x, double a,
                            int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return static_cast<int>(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

__global__ void reset_kernel(int* flags, int64_t nf, int* counter, int* extra, int64_t ne) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < nf; i += stride) flags[i] = 0;
  for (int64_t i = i0; i < ne; i += stride) extra[i] = 0;
  if (i0 == 0) counter[0] = 0;
}

struct PackBounds {
  int b[kMaxPackRanks + 1];
};

// threadIdx.x runs over the n0 columns (coalesced on the run side, and on the
// segment side within a segment), threadIdx.y and the grid over the runs; a
// thread's columns keep their segment, so the segment lookup is outside the
// row loop.
template <bool UNPACK>
__global__ void __launch_bounds__(256) slab_pack_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                                        int64_t rows, int n0, int nranks, PackBounds pb) {
  const int64_t rstep = static_cast<int64_t>(gridDim.x) * blockDim.y;
  for (int i0 = threadIdx.x; i0 < n0; i0 += blockDim.x) {
    int q = 0;
    while (q + 1 < nranks && i0 >= pb.b[q + 1]) ++q;
    const int w = pb.b[q + 1] - pb.b[q];
    const int64_t seg = rows * pb.b[q] + (i0 - pb.b[q]);
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.y + threadIdx.y; r < rows; r += rstep) {
      if (UNPACK) dst[r * n0 + i0] = src[seg + r * w];
      else dst[seg + r * w] = src[r * n0 + i0];
    }
  }
}

}  // namespace

cudaError_t slab_pack(const double* src, double* dst, int64_t rows, int n0, int nranks, const int* b0,
                      int dir, cudaStream_t st) {
  if (rows <= 0 || n0 <= 0) return cudaSuccess;
  if (nranks < 1 || nranks > kMaxPackRanks || b0[0] != 0 || b0[nranks] != n0) return cudaErrorInvalidValue;
  PackBounds pb{};
  for (int q = 0; q <= nranks; ++q) pb.b[q] = b0[q];
  int bx = 32;
  while (bx < n0 && bx < 256) bx *= 2;
  const dim3 block(bx, 256 / bx);
  const int64_t want = (rows + block.y - 1) / block.y;
  const int grid = static_cast<int>(std::min<int64_t>(want, 148 * 8));
  if (dir) slab_pack_kernel<true><<<grid, block, 0, st>>>(src, dst, rows, n0, nranks, pb);
  else slab_pack_kernel<false><<<grid, block, 0, st>>>(src, dst, rows, n0, nranks, pb);
  return cudaGetLastError();
}

cudaError_t reset_state(int* flags, int64_t nf, int* counter, int* extra, int64_t ne, cudaStream_t st) {
  const int64_t n = nf > ne ? nf : ne;
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256 + 1, 1184));
  reset_kernel<<<blocks, 256, 0, st>>>(flags, nf, counter, extra, extra ? ne : 0);
  return cudaGetLastError();
}

cudaError_t sumsq(const double* x, int64_t n, double* out_dev, cudaStream_t st) {
  sumsq_kernel<<<grid_for(n), 256, 0, st>>>(x, n, out_dev);
  return cudaGetLastError();
}

cudaError_t axpy(double* y, const double* x, double a, int64_t n, cudaStream_t st) {
  axpy_kernel<<<grid_for(n), 256, 0, st>>>(y, x, a, n);
  return cudaGetLastError();
}

}  // namespace tsg

namespace tsg {

cudaError_t kernel_setup(const void* fn, size_t smem, int threads, int* nsm, int* occ) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> attr;           // (fn, dev) -> opt-in
  static std::map<std::tuple<const void*, int, size_t, int>, int> occs;  // -> CTAs per SM
  static std::map<int, int> sms;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  int& ns = sms[dev];
  if (!ns) {
    e = cudaDeviceGetAttribute(&ns, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
  }
  size_t& at = attr[{fn, dev}];
  if (smem > at || (smem > 0 && at == 0)) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    at = smem;
  }
  int& oc = occs[{fn, dev, smem, threads}];
  if (!oc) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, fn, threads, smem);
    if (e != cudaSuccess) return e;
    if (oc < 1) return cudaErrorInvalidConfiguration;
  }
  *nsm = ns;
  *occ = oc;
  return cudaSuccess;
}

}  // namespace tsg
