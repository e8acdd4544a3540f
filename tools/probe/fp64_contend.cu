// Does a DMMA stream on other warps slow a DFMA dependency chain?  Warp 0:
// DFMA chain (cycles/op); warps 1..W-1: DMMA loops on the same or other
// sub-partitions (warp w sits on SMSP w % 4).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, int dmma_warps_mask) {
  const int w = threadIdx.x >> 5;
  double x = 1.0 + threadIdx.x * 1e-9, y = 1.0000001;
  if (w == 0) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
  } else if ((dmma_warps_mask >> w) & 1) {
    double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < 4 * n; ++i) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[2 * j]), "+d"(c[2 * j + 1]) : "d"(y), "d"(x));
    }
    x = c[0] + c[1] + c[2] + c[3] + c[4] + c[5] + c[6] + c[7];
  }
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64 * 8);
  const int n = 2000;
  struct { const char* name; int mask; } cases[] = {
      {"alone", 0}, {"DMMA on other SMSPs (warps 1,2,3)", 0xE}, {"DMMA on same SMSP (warp 4)", 0x10},
      {"DMMA on same SMSP (warps 4,8,12)", 0x1110}, {"DMMA everywhere (warps 1..15)", 0xFFFE}};
  for (auto& cs : cases) {
    k<<<1, 512>>>(o, c, n, cs.mask);
    k<<<1, 512>>>(o, c, n, cs.mask);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-40s DFMA chain %.1f cycles/op\n", cs.name, double(h) / n);
  }
  return 0;
}
