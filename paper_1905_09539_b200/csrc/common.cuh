// Shared device helpers for the sm_100a FP64 kernels.
//
// FP64 on Blackwell has no tcgen05 kind (ptxas rejects .kind::f64, SURVEY
// §2.3), so the tensor-core path is warp-level mma.sync m8n8k4 f64, which
// ptxas lowers to SASS DMMA.8x8x4 (measured 37.07 TFLOP/s/GPU peak,
// profiles/r01_fp64_peak_probe.log).  Operands are staged global -> shared
// with cp.async (LDGSTS) multi-stage pipelines.
#pragma once
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

#define TSG_DEVINL __device__ __forceinline__

namespace tsg {

// D = A(8x4, row) * B(4x8, col) + C(8x8).  Fragment ownership per lane
// (g = lane>>2, t = lane&3):  a = A[g][t], b = B[t][g], c = C[g][2t..2t+1].
#ifndef TSG_DMMA_VOLATILE
#define TSG_DMMA_VOLATILE 1
#endif
TSG_DEVINL void dmma(double& c0, double& c1, double a, double b) {
#if TSG_DMMA_VOLATILE
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
#else
  // no side effects: let the compiler schedule the products freely
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
#endif
}

TSG_DEVINL uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async copy, L2-only (.cg); src_bytes < 16 zero-fills the rest.
TSG_DEVINL void cp_async16(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(src_bytes));
}
// 8-byte async copy (.ca: 4/8-byte copies cannot use .cg).
TSG_DEVINL void cp_async8(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(src_bytes));
}
TSG_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
TSG_DEVINL void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
TSG_DEVINL void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// Acquire/release flag primitives for the dataflow solver (gpu scope).
TSG_DEVINL int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
TSG_DEVINL void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// Programmatic dependent launch trigger: lets the next kernel in the stream
// (a tile-flag-gated back transform) launch while this grid still runs.
TSG_DEVINL void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
// Wait for the preceding grid's completion and memory flush when this grid was
// launched as a programmatic dependent (returns at once otherwise).
TSG_DEVINL void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Host: launch `k` as a programmatic dependent of the previous kernel in `st`
// (it may start once every CTA of that kernel has called pdl_trigger(); the
// kernel must call pdl_wait() before touching the predecessor's outputs).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
// System scope (tiles and flags shared with peer GPUs over NVLink).
TSG_DEVINL int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
TSG_DEVINL void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// Uncached (volatile) load for peer-written tiles.
TSG_DEVINL double ld_volatile(const double* p) {
  double v;
  asm volatile("ld.volatile.global.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}
TSG_DEVINL double ld_cg(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}

}  // namespace tsg
