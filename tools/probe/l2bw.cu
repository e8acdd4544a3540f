// L2 / HBM read bandwidth probe: every SM streams a buffer of `bytes`
// (fits L2 when small) `reps` times with 16-byte loads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double2* __restrict__ p, size_t n, int reps, double* out) {
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(p + ((i + r * 977) % n));
      s += v.x + v.y;
    }
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* out; cudaMalloc(&out, 8);
  for (size_t mb : {16, 32, 64, 96, 512, 2048}) {
    size_t bytes = mb << 20, n = bytes / 16;
    double2* p; cudaMalloc(&p, bytes); cudaMemset(p, 0, bytes);
    int reps = mb <= 96 ? 20 : 3;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    rd<<<148 * 8, 512>>>(p, n, 1, out);
    cudaEventRecord(a);
    rd<<<148 * 8, 512>>>(p, n, reps, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%5zu MB x%d: %.1f GB/s\n", mb, reps, (double)bytes * reps / ms / 1e6);
    cudaFree(p);
  }
  return 0;
}
