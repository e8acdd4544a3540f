// Latency of the fibre-solve leader's in-block substitution (sub8 x 2 +
// the 8x8 coupling) on one warp alone: cycles per super-block step.
#include "../../paper_1905_09539_b200/csrc/solve_fibre.cu"
#include <cstdio>
namespace tsg {
template <bool PRO>
__global__ void leader_probe(const FibreArgs a, double* Y, long long* cyc, int steps, unsigned code_lo, unsigned code_hi) {
  __shared__ double Td[192];
  for (int e = threadIdx.x; e < 192; e += 32) Td[e] = (e % 9 == 0) ? 3.0 : 0.01 * (e % 7);
  __syncwarp();
  const int lane = threadIdx.x;
  const int pitch = 36;
  const int mycol = lane < 16 ? lane : -1;
  const int role = lane < 16 ? (lane & 1) : 3;
  const int partner = role == 0 ? lane + 1 : role == 1 ? lane - 1 : lane;
  const double sgn = role == 1 ? -1.0 : 1.0, mysr = 0.5, mysi = 0.25;
  const double t2 = 1e-30;
  long long t0 = clock64();
  bool bad = false;
  for (int q = 0; q < steps; ++q) {
    double zl[8], zh[8];
    const bool own = mycol >= 0;
    const int nl = 8, nh = 8, i0 = (q & 15) * 16, mid = i0 + 8;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      zl[r] = (own && r < nl) ? Y[(i0 + r) * pitch + mycol] : 0.0;
      zh[r] = (own && r < nh) ? Y[(mid + r) * pitch + mycol] : 0.0;
    }
    const double* T3 = Td;
    bad = sub8<PRO>(zh, nh, code_hi, partner, sgn, mysr, mysi, t2, T3 + 64) || bad;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      double acc = zl[r];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc = fma(-T3[128 + r * 8 + k], zh[k], acc);
      zl[r] = acc;
    }
    bad = sub8<PRO>(zl, PRO ? nl : 8, PRO ? code_lo : 0u, partner, sgn, mysr, mysi, t2, T3) || bad;
    if (own) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        Y[(i0 + r) * pitch + mycol] = zl[r];
        Y[(mid + r) * pitch + mycol] = zh[r];
      }
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[0] = t1 - t0;
  if (bad) cyc[1] = 1;
}
}  // namespace tsg
int main() {
  double* Y; long long* c; cudaMalloc(&Y, 256 * 36 * 8); cudaMalloc(&c, 16);
  cudaMemset(Y, 0, 256 * 36 * 8);
  tsg::FibreArgs a{};
  a.tiny = 1e-15;
  const int steps = 1000;
  struct { const char* n; unsigned lo, hi; } cs[] = {{"all 1x1", 0u, 0u}, {"all 2x2", 0x9999u, 0x9999u}};
  for (int pro = 0; pro < 2; ++pro)
  for (auto& x : cs) {
    for (int r = 0; r < 2; ++r) {
      if (pro) tsg::leader_probe<true><<<1, 32, 0>>>(a, Y, c, steps, x.lo, x.hi);
      else tsg::leader_probe<false><<<1, 32, 0>>>(a, Y, c, steps, x.lo, x.hi);
    }
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%s %-10s %.0f cycles per 16-row step\n", pro ? "prologue (runtime code)" : "chain, compile-time all-1x1 code", x.n, double(h) / steps);
  }
  return 0;
}
