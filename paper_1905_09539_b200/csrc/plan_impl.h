// Internal declarations shared by plan.cpp (single-GPU plans) and dist.cpp
// (slab-sharded multi-GPU plans).  Not part of the C-ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tsylv_gpu.h"
#include "solve.h"

struct tsg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  cudaEvent_t ev[8] = {};
};

struct DevBuf {
  double* p = nullptr;
  size_t n = 0;
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  cudaError_t ensure(size_t count) {
    if (count <= n) return cudaSuccess;
    reset();
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(double));
    if (e == cudaSuccess) n = count;
    return e;
  }
  ~DevBuf() { reset(); }
};

// Launch-order and diagnostic switches, fixed when the plan is created.
// serial: every kernel after its predecessor (tsg_plan_set_serial; env
// TSG_GATE=0 at creation), schain_off: no slab chain between the first two
// transform GEMMs (TSG_SCHAIN=0), verbose: one line per solve on stderr
// (TSG_VERBOSE).  The development probes (trace, prof, dbg: per-hyperplane
// release times, per-phase cycle counters, kernel ablations) are read only
// in a -DTSG_DEVTOOLS build (tools/README.md); the shipped library never
// reads them.
struct PlanKnobs {
  bool serial = false, schain_off = false, verbose = false;
  bool trace = false, prof = false, dbg_fdone = false;
  int dbg = 0;
  static PlanKnobs from_env();
};

struct tsg_plan {
  tsg_ctx* ctx = nullptr;
  PlanKnobs knobs;
  int skip_mask = 0;   // modes with identity transforms (tsg_opts::skip_transform_mask)
  int force_f = -1;    // decoupled free mode (tsg_opts::free_mode)
  int family = 0, d = 0, reduced_only = 0;
  std::vector<int> dims;
  std::vector<int64_t> stride;
  int64_t N = 0;
  // device factors
  std::vector<DevBuf> T, Fwd, FwdT, Bwd, BwdT, eig, pdat, dhat, vhat;  // per mode
  DevBuf Tc;
  std::vector<tsg::TileMode*> tmode;
  std::vector<int*> bnd;
  std::vector<int*> rowtile;  // per mode: tile index of every row
  int* order = nullptr;
  unsigned long long* ocoord = nullptr;
  int fast = 0;  // 1: solve_lap_kernel, 3: solve_lap3_kernel (Laplace, good eigenbases)
  int lt3 = 3;   // log2 tile extent of solve_lap3
  bool use16 = false;  // 16^3 TMA kernel (solve_lap16.cu)
  std::vector<int> tlog, tsh;  // solve_lapd padded tile layout
  int* flags = nullptr;
  int* counter = nullptr;   // [0] = queue head, [1] = status
  // Back transform mode 0 gated on tile flags and launched as a programmatic
  // dependent of the solve (overlaps the solve's drain): per 64-column group
  // of X_(0), the linear ids of the tiles (0, t_1, .., t_{d-1}) it reads.
  int* gate_off = nullptr;
  int* gate_ids = nullptr;
  int gate_groups = 0;
  // Slab chain between the mode-0 and mode-1 transform GEMMs (fwd, back):
  // done flags of the mode-0 GEMM's CTA tiles (s_tm m-tiles, width s_bn),
  // one allocation (sdone[1] = sdone[0] + sdone_n) reset at every solve.
  int* sdone[2] = {nullptr, nullptr};
  int sdone_n = 0, s_tm = 0, s_bn = 0;
  // Trailing cube (lap16d): the last `cube` tiles of every mode are solved
  // by a small first grid (cube_grid CTAs, own queue) that runs beside the
  // last forward GEMM, gated per tile on that GEMM's done flags (fdone);
  // the main grid takes the other tiles.  aux = [sdone fwd | sdone back |
  // fdone | cube queue head], reset with the tile flags at every solve.
  int cube = 0, cube_grid = 0;
  int* order1 = nullptr;
  int* order2 = nullptr;
  unsigned long long* ocoord1 = nullptr;
  unsigned long long* ocoord2 = nullptr;
  int64_t ntiles1 = 0, ntiles2 = 0;
  int* fdone = nullptr;
  int fdone_n = 0, fg_bm = 0, fg_bn = 0, fg_tm = 0;
  int* aux = nullptr;
  int64_t aux_n = 0;
  int64_t ntiles = 0;
  std::vector<std::vector<int>> bds_h;  // host tile boundaries per mode
  std::vector<int> order_h;             // host topological order (linear tile ids)
  std::vector<int> ntiles_mode, tile_ext;
  // work buffers
  DevBuf xdev, w1, w2;
  DevBuf sin[2], sout[2];  // tsg_plan_execute_stream staging (double-buffered)
  std::vector<DevBuf> wchain;  // gsylv W_m, m = 1..d-1
  double flops_alg = 0, flops_exec = 0;
  double tiny = 0;
  double max_cond = 0;  // worst 2x2 eigenbasis condition (Frobenius)
  int refine = 0;
  tsg::SolveLaunchInfo solve_info{};
  // Eigen-decoupled fibre solve (decouple.cpp, solve_fibre.cu): modes other
  // than `dec_f` are folded into their eigenbases by the transforms.
  int decoupled = 0, dec_f = -1;
  double dec_kappa = 0;
  tsg::FibreArgs fib{};
  std::vector<void*> owned;  // device tables of the fibre solve
  // graph cache
  cudaGraphExec_t gexec = nullptr;
  const double* g_in = nullptr;
  double* g_out = nullptr;
  int launches = 0;
  ~tsg_plan() {
    for (auto* b : tmode)
      if (b) cudaFree(b);
    for (auto* b : bnd)
      if (b) cudaFree(b);
    for (auto* b : rowtile)
      if (b) cudaFree(b);
    if (order) cudaFree(order);
    if (ocoord) cudaFree(ocoord);
    if (flags) cudaFree(flags);
    if (counter) cudaFree(counter);
    if (gate_off) cudaFree(gate_off);
    if (gate_ids) cudaFree(gate_ids);
    if (aux) cudaFree(aux);
    for (void* q : {static_cast<void*>(order1), static_cast<void*>(order2), static_cast<void*>(ocoord1),
                    static_cast<void*>(ocoord2)})
      if (q) cudaFree(q);
    if (gexec) cudaGraphExecDestroy(gexec);
    for (void* q : owned)
      if (q) cudaFree(q);
  }
};


namespace tsg_impl {

// set while tsg_dplan_create builds its plan (the sharded solve runs the 8^3 kernel)
extern thread_local bool g_force_lap3;

int fail(tsg_ctx* ctx, int code, const std::string& msg);
cudaError_t upload_mat(DevBuf& b, const double* h, size_t n);
std::vector<double> transpose(const double* a, int n);
// Solve arguments of a plan over work tensor `work` (everything except the
// queue, flags and status fields).
void fill_solve_args(const tsg_plan* pl, double* work, tsg::SolveArgs& a);
// Launch the plan's dataflow kernel with fully populated arguments.
cudaError_t launch_plan_solve(tsg_plan* pl, const tsg::SolveArgs& a, cudaStream_t st);
// Tile boundaries of a mode (2x2 Schur blocks never split).
std::vector<int> tile_bounds_of(const double* T, int n, int b);

}  // namespace tsg_impl

#define TSG_CU(call)                                                                 \
  do {                                                                               \
    cudaError_t _e = (call);                                                         \
    if (_e != cudaSuccess)                                                           \
      return tsg_impl::fail(ctx, TSG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)
