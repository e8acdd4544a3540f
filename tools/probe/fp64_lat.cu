// Dependent-chain latencies on one warp (cycles per op): DFMA, DADD, DMUL,
// FP64 division, double __shfl_sync, DMMA m8n8k4 (accumulator chain), LDS.64.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double x0, int n) {
  __shared__ double sm[64];
  double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0, t1;
  sm[threadIdx.x] = x;
  __syncwarp();
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  double c0 = x, c1 = y;
  t0 = clock64();
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(y), "d"(x));
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { x = sm[idx]; idx = (static_cast<int>(x) & 31); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = t1 - t0;
  out[threadIdx.x] = x + c0 + c1;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 64 * 8);
  const int n = 1000;
  lat<<<1, 32>>>(o, c, 1.0, n);
  lat<<<1, 32>>>(o, c, 1.0, n);
  long long h[8]; cudaMemcpy(h, c, 7 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"DFMA", "DADD", "DMUL", "div 1/(x+1)", "shfl double", "DMMA chain", "LDS dep"};
  for (int i = 0; i < 7; ++i) printf("%-14s %.1f cycles/op\n", nm[i], double(h[i]) / n);
  return 0;
}
