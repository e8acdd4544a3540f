// Probe TMA (cp.async.bulk.tensor) alignment rules for FP64 3D boxes.
#include <cstdio>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_1905_09539_b200/csrc/tma.h"

__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, int soff, double* out, unsigned bytes) {
  extern __shared__ __align__(1024) double sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { tsg::mbar_init(&bar, 1); tsg::mbar_fence_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    tsg::mbar_expect_tx(&bar, bytes);
    tsg::tma_load_3d(sm + soff, &m, c0, c1, c2, &bar);
  }
  tsg::mbar_wait(&bar, 0);
  if (threadIdx.x == 0) out[0] = sm[soff];
}

int main() {
  double* x; cudaMalloc(&x, 8 * 3 * 8 * 8);
  double* out; cudaMalloc(&out, 8);
  const uint64_t dims[3] = {8, 3, 8};
  for (int m = 0; m < 3; ++m) {
    uint32_t box[3] = {8, 8, 8};
    box[m] = 32;
    CUtensorMap mp;
    printf("m=%d encode %d\n", m, (int)tsg::encode_tmap_f64(&mp, x, 3, dims, box));
    int cs[][3] = {{0, 0, 0}, {4, 0, 0}, {6, 2, 4}, {0, 2, 6}, {2, 0, 4}};
    for (auto& c : cs) {
      k<<<1, 32, 70000>>>(mp, c[0], c[1], c[2], 0, out, 8 * 8 * 32 * 8);
      cudaError_t e = cudaDeviceSynchronize();
      printf("  c=(%d,%d,%d): %s\n", c[0], c[1], c[2], cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
