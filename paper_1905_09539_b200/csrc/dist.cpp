// Slab-sharded multi-GPU plans (include/tsylv_gpu.h, tsg_dplan_*).
//
// the tensor is partitioned into slabs along its last mode
// (tile-aligned, so no slab boundary cuts a 2x2 Schur block -- the
// split_index rule of the reference, sylvester.hpp:43-49).  Transforms along
// modes 0..d-2 are slab-local; the last-mode transform needs every slab and
// runs as an all-gather (NCCL, issued by the caller between the _local and
// _split steps) followed by one rectangular DMMA GEMM per slab against the
// zero-padded rows of U_{d-1}^T (forward) or U_{d-1} (back).
//
// The reduced solve is the single-GPU dataflow kernel (solve_lap3.cu) run on
// every GPU over its own tiles, with the tiles of the other slabs and their
// release flags read through CUDA IPC peer mappings (NVLink):
// system-scope release after a tile is scattered, system-scope acquire
// before it is read, volatile loads for peer tile data.  Flags carry an
// epoch per solve, so no rank ever resets a flag another rank may read.
// In emulated mode one process owns every slab (separate buffers) on one
// GPU and launches one kernel over all tiles: the same addressing and
// queue logic, provably free of cross-launch waits (B200_PROFILING.md).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/tsylv_gpu.h"
#include "gemm.h"
#include "plan_impl.h"
#include "util.h"
#include "solve.h"

using tsg_impl::fail;
using tsg_impl::upload_mat;

struct tsg_dplan {
  tsg_ctx* ctx = nullptr;
  int rank = 0, nranks = 1, emulate = 0, d = 0;
  std::vector<int> dims;
  int64_t plane = 1;  // elements of one last-mode row (prod dims[0..d-2])
  std::vector<int> slo;  // nranks + 1
  int rmax = 0;
  tsg_plan* pl = nullptr;  // reduced plan over the full dims (tile tables)
  std::vector<DevBuf> xs;  // slab tensors (all slabs emulated, own slab otherwise)
  DevBuf send, gath, tmp;
  std::vector<DevBuf> fwd, fwdT, bwd, bwdT;  // local modes 0..d-2
  std::vector<DevBuf> af, afT, ab, abT;      // last mode, per owned slab (padded)
  // multi-GPU peers
  double* peer_x[tsg::kMaxSlabs] = {};
  int* peer_f[tsg::kMaxSlabs] = {};
  int* order_own = nullptr;
  unsigned long long* ocoord_own = nullptr;
  int64_t ntiles_own = 0;
  int epoch = 0;
  ~tsg_dplan() {
    for (int q = 0; q < tsg::kMaxSlabs; ++q) {
      if (peer_x[q]) cudaIpcCloseMemHandle(peer_x[q]);
      if (peer_f[q]) cudaIpcCloseMemHandle(peer_f[q]);
    }
    if (order_own) cudaFree(order_own);
    if (ocoord_own) cudaFree(ocoord_own);
    if (pl) tsg_plan_destroy(pl);
  }
  int rows(int q) const { return slo[q + 1] - slo[q]; }
  bool owns(int q) const { return emulate || q == rank; }
  std::vector<int> slab_dims(int q) const {
    std::vector<int> v = dims;
    v[d - 1] = rows(q);
    return v;
  }
};

namespace {

cudaStream_t pick(tsg_dplan* dp, void* stream) {
  return stream ? static_cast<cudaStream_t>(stream) : dp->ctx->stream;
}

// Balanced, tile-aligned split of the tile boundaries `bd` into k slabs.
std::vector<int> split_tiles(const std::vector<int>& bd, int k) {
  const int nt = static_cast<int>(bd.size()) - 1;
  std::vector<int> out{0};
  for (int q = 1; q < k; ++q) {
    // first tile boundary at or after the ideal row q * n / k
    // nearest tile boundary to the ideal row q * n / k (strictly increasing)
    const double ideal = static_cast<double>(bd[nt]) * q / k;
    int best = -1;
    for (int t = 1; t < nt; ++t) {
      if (bd[t] <= out.back()) continue;
      if (best < 0 || std::abs(bd[t] - ideal) < std::abs(bd[best] - ideal)) best = t;
    }
    out.push_back(best < 0 ? bd[nt] : bd[best]);
  }
  out.push_back(bd[nt]);
  return out;
}

double* vbase(double* p, int lo, int64_t plane) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(p) -
                                   static_cast<int64_t>(lo) * plane * static_cast<int64_t>(sizeof(double)));
}

}  // namespace

extern "C" {

int tsg_slab_bounds(int n, const double* T, int tile, int nranks, int* bounds) {
  if (n <= 0 || !T || tile <= 0 || nranks <= 0 || nranks > tsg::kMaxSlabs || !bounds) return TSG_EINVAL;
  const std::vector<int> bd = tsg_impl::tile_bounds_of(T, n, tile);
  if (static_cast<int>(bd.size()) - 1 < nranks) return TSG_EDIM;  // fewer tiles than ranks
  const std::vector<int> s = split_tiles(bd, nranks);
  for (int q = 0; q <= nranks; ++q) bounds[q] = s[q];
  for (int q = 0; q < nranks; ++q)
    if (bounds[q + 1] <= bounds[q]) return TSG_EDIM;
  return TSG_OK;
}

int tsg_slab_pack(tsg_ctx* ctx, const double* src, double* dst, long long rows, int n0, int nranks,
                  const int* b0, int dir, void* stream) {
  if (!ctx || !src || !dst || !b0 || rows < 0 || n0 <= 0) return TSG_EINVAL;
  if (nranks < 1 || nranks > tsg::kMaxPackRanks || b0[0] != 0 || b0[nranks] != n0)
    return fail(ctx, TSG_EINVAL, "slab_pack: bounds must run from 0 to n0 over at most 64 ranks");
  for (int q = 0; q < nranks; ++q)
    if (b0[q + 1] < b0[q]) return fail(ctx, TSG_EINVAL, "slab_pack: bounds must be non-decreasing");
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  TSG_CU(tsg::slab_pack(src, dst, rows, n0, nranks, b0, dir != 0, st));
  return TSG_OK;
}

int tsg_dplan_create(tsg_ctx* ctx, int rank, int nranks, int emulate, int d, const int* dims,
                     const double* const* T, const double* const* U, const tsg_opts* opts,
                     tsg_dplan** out) {
  if (!ctx || !out) return TSG_EINVAL;
  *out = nullptr;
  if (nranks < 1 || nranks > tsg::kMaxSlabs || rank < 0 || rank >= nranks)
    return fail(ctx, TSG_EINVAL, "dplan: rank/nranks out of range (at most 8 slabs)");
  if (d != 3) return fail(ctx, TSG_EDIM, "dplan: the sharded solve supports order d = 3");
  for (int m = 0; m < d; ++m)
    if (!U[m]) return fail(ctx, TSG_EDIM, "dplan: missing orthogonal factor");
  auto dp = std::make_unique<tsg_dplan>();
  dp->ctx = ctx;
  dp->rank = rank;
  dp->nranks = nranks;
  dp->emulate = emulate ? 1 : 0;
  dp->d = d;
  dp->dims.assign(dims, dims + d);
  for (int m = 0; m < d - 1; ++m) dp->plane *= dims[m];
  tsg_impl::g_force_lap3 = true;
  int rc = tsg_plan_create(ctx, 0, d, dims, T, nullptr, nullptr, nullptr, 1, opts, &dp->pl);
  tsg_impl::g_force_lap3 = false;
  if (rc != TSG_OK) return rc;
  tsg_plan* pl = dp->pl;
  if (pl->fast != 3 || pl->lt3 != 3)
    return fail(ctx, TSG_EINVAL, "dplan: needs the order-3 Laplace fast path (8^3 tiles)");
  pl->w1.reset();  // the slabs replace the plan's work tensor
  TSG_CU(cudaSetDevice(ctx->device));
  const int n = dims[d - 1];
  const std::vector<int>& bd = pl->bds_h[d - 1];
  if (static_cast<int>(bd.size()) - 1 < nranks)
    return fail(ctx, TSG_EDIM, "dplan: fewer tiles along the last mode than ranks");
  dp->slo = split_tiles(bd, nranks);
  for (int q = 0; q < nranks; ++q) {
    if (dp->rows(q) <= 0) return fail(ctx, TSG_EDIM, "dplan: empty slab");
    dp->rmax = std::max(dp->rmax, dp->rows(q));
  }
  const int64_t P = nranks, rm = dp->rmax, K = P * rm;
  // slabs
  dp->xs.resize(nranks);
  for (int q = 0; q < nranks; ++q)
    if (dp->owns(q)) TSG_CU(dp->xs[q].ensure(static_cast<size_t>(dp->rows(q)) * dp->plane));
  // gather (+ send in multi-GPU mode), padding rows zeroed once (never written)
  TSG_CU(dp->gath.ensure(static_cast<size_t>(K) * dp->plane));
  TSG_CU(cudaMemset(dp->gath.p, 0, static_cast<size_t>(K) * dp->plane * sizeof(double)));
  if (!dp->emulate) {
    TSG_CU(dp->send.ensure(static_cast<size_t>(rm) * dp->plane));
    TSG_CU(cudaMemset(dp->send.p, 0, static_cast<size_t>(rm) * dp->plane * sizeof(double)));
  }
  TSG_CU(dp->tmp.ensure(static_cast<size_t>(rm) * dp->plane));
  // local-mode factors
  dp->fwd.resize(d - 1);
  dp->fwdT.resize(d - 1);
  dp->bwd.resize(d - 1);
  dp->bwdT.resize(d - 1);
  for (int m = 0; m < d - 1; ++m) {
    const size_t nn = static_cast<size_t>(dims[m]) * dims[m];
    const std::vector<double> ut = tsg_impl::transpose(U[m], dims[m]);
    TSG_CU(upload_mat(dp->fwd[m], ut.data(), nn));
    TSG_CU(upload_mat(dp->fwdT[m], U[m], nn));
    TSG_CU(upload_mat(dp->bwd[m], U[m], nn));
    TSG_CU(upload_mat(dp->bwdT[m], ut.data(), nn));
  }
  // last-mode factors per owned slab: rows R_q of U^T (forward) / U (back),
  // columns scattered to the padded gather layout (slab q' at q' * rmax)
  dp->af.resize(nranks);
  dp->afT.resize(nranks);
  dp->ab.resize(nranks);
  dp->abT.resize(nranks);
  const double* Ul = U[d - 1];
  for (int q = 0; q < nranks; ++q) {
    if (!dp->owns(q)) continue;
    const int r = dp->rows(q);
    std::vector<double> f(static_cast<size_t>(r) * K, 0.0), fT(f.size(), 0.0), b(f.size(), 0.0),
        bT(f.size(), 0.0);
    for (int qq = 0; qq < nranks; ++qq)
      for (int j = 0; j < dp->rows(qq); ++j) {
        const int64_t col = qq * rm + j, gj = dp->slo[qq] + j;
        for (int i = 0; i < r; ++i) {
          const int64_t gi = dp->slo[q] + i;
          const double ut = Ul[gj + gi * n];  // U^T[gi][gj] = U[gj][gi]
          const double u = Ul[gi + gj * n];   // U[gi][gj]
          f[i + col * r] = ut;
          fT[col + static_cast<int64_t>(i) * K] = ut;
          b[i + col * r] = u;
          bT[col + static_cast<int64_t>(i) * K] = u;
        }
      }
    TSG_CU(upload_mat(dp->af[q], f.data(), f.size()));
    TSG_CU(upload_mat(dp->afT[q], fT.data(), fT.size()));
    TSG_CU(upload_mat(dp->ab[q], b.data(), b.size()));
    TSG_CU(upload_mat(dp->abT[q], bT.data(), bT.size()));
  }
  // tiles of this rank (all tiles when emulated), topological order kept
  {
    std::vector<int> ord;
    std::vector<unsigned long long> oc;
    const std::vector<int>& nt = pl->ntiles_mode;
    const int64_t lastmul = static_cast<int64_t>(nt[0]) * nt[1];
    for (int t : pl->order_h) {
      const int t2 = static_cast<int>(t / lastmul);
      const int row = bd[t2];
      int q = 0;
      while (q + 1 < nranks && row >= dp->slo[q + 1]) ++q;
      if (!dp->owns(q)) continue;
      ord.push_back(t);
      int64_t r = t;
      unsigned long long pk = 0;
      for (int m = 0; m < d; ++m) {
        pk |= static_cast<unsigned long long>(r % nt[m]) << (10 * m);
        r /= nt[m];
      }
      oc.push_back(pk);
    }
    dp->ntiles_own = static_cast<int64_t>(ord.size());
    TSG_CU(cudaMalloc(&dp->order_own, std::max<size_t>(ord.size(), 1) * sizeof(int)));
    TSG_CU(cudaMemcpy(dp->order_own, ord.data(), ord.size() * sizeof(int), cudaMemcpyHostToDevice));
    TSG_CU(cudaMalloc(&dp->ocoord_own, std::max<size_t>(oc.size(), 1) * sizeof(unsigned long long)));
    TSG_CU(cudaMemcpy(dp->ocoord_own, oc.data(), oc.size() * sizeof(unsigned long long),
                      cudaMemcpyHostToDevice));
  }
  TSG_CU(cudaMemset(pl->flags, 0, pl->ntiles * sizeof(int)));  // epoch 0
  TSG_CU(cudaDeviceSynchronize());
  *out = dp.release();
  return TSG_OK;
}

void tsg_dplan_destroy(tsg_dplan* dp) { delete dp; }

int tsg_dplan_info(const tsg_dplan* dp, int* bounds, int64_t* slab_elems, int64_t* send_elems) {
  if (!dp) return TSG_EINVAL;
  if (bounds)
    for (int q = 0; q <= dp->nranks; ++q) bounds[q] = dp->slo[q];
  if (slab_elems) *slab_elems = static_cast<int64_t>(dp->rows(dp->rank)) * dp->plane;
  if (send_elems) *send_elems = static_cast<int64_t>(dp->rmax) * dp->plane;
  return TSG_OK;
}

int tsg_dplan_buffers(tsg_dplan* dp, double** send, double** gather) {
  if (!dp) return TSG_EINVAL;
  if (send) *send = dp->emulate ? nullptr : dp->send.p;
  if (gather) *gather = dp->gath.p;
  return TSG_OK;
}

int tsg_dplan_ipc_export(tsg_dplan* dp, void* handles) {
  if (!dp || !handles) return TSG_EINVAL;
  tsg_ctx* ctx = dp->ctx;
  if (dp->emulate) return fail(ctx, TSG_EINVAL, "dplan: no IPC in emulated mode");
  static_assert(2 * sizeof(cudaIpcMemHandle_t) == TSG_IPC_BYTES, "IPC handle size");
  auto* h = static_cast<cudaIpcMemHandle_t*>(handles);
  TSG_CU(cudaIpcGetMemHandle(&h[0], dp->xs[dp->rank].p));
  TSG_CU(cudaIpcGetMemHandle(&h[1], dp->pl->flags));
  return TSG_OK;
}

int tsg_dplan_ipc_import(tsg_dplan* dp, const void* all_handles) {
  if (!dp || !all_handles) return TSG_EINVAL;
  tsg_ctx* ctx = dp->ctx;
  if (dp->emulate) return fail(ctx, TSG_EINVAL, "dplan: no IPC in emulated mode");
  TSG_CU(cudaSetDevice(ctx->device));
  const auto* h = static_cast<const cudaIpcMemHandle_t*>(all_handles);
  for (int q = 0; q < dp->nranks; ++q) {
    if (q == dp->rank || dp->peer_x[q]) continue;
    void* px = nullptr;
    void* pf = nullptr;
    TSG_CU(cudaIpcOpenMemHandle(&px, h[2 * q], cudaIpcMemLazyEnablePeerAccess));
    TSG_CU(cudaIpcOpenMemHandle(&pf, h[2 * q + 1], cudaIpcMemLazyEnablePeerAccess));
    dp->peer_x[q] = static_cast<double*>(px);
    dp->peer_f[q] = static_cast<int*>(pf);
  }
  return TSG_OK;
}

int tsg_dplan_forward_local(tsg_dplan* dp, const double* B, void* stream) {
  if (!dp || !B) return TSG_EINVAL;
  tsg_ctx* ctx = dp->ctx;
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = pick(dp, stream);
  const int d = dp->d;
  for (int q = 0; q < dp->nranks; ++q) {
    if (!dp->owns(q)) continue;
    const std::vector<int> sd = dp->slab_dims(q);
    const double* src = dp->emulate ? B + static_cast<int64_t>(dp->slo[q]) * dp->plane : B;
    double* dst_final = dp->emulate ? dp->gath.p + static_cast<int64_t>(q) * dp->rmax * dp->plane : dp->send.p;
    // modes 0..d-2, ping-pong ending in the send slot
    for (int m = 0; m < d - 1; ++m) {
      double* dst = ((d - 2 - m) % 2 == 0) ? dst_final : dp->tmp.p;
      TSG_CU(tsg::mode_product(src, dst, d, sd.data(), m, dp->fwd[m].p, dp->fwdT[m].p, sd[m], 1.0, 0.0, st));
      src = dst;
    }
  }
  return TSG_OK;
}

int tsg_dplan_forward_split(tsg_dplan* dp, void* stream) {
  if (!dp) return TSG_EINVAL;
  tsg_ctx* ctx = dp->ctx;
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = pick(dp, stream);
  std::vector<int> gd = dp->dims;
  gd[dp->d - 1] = dp->nranks * dp->rmax;
  for (int q = 0; q < dp->nranks; ++q) {
    if (!dp->owns(q)) continue;
    TSG_CU(tsg::mode_product(dp->gath.p, dp->xs[q].p, dp->d, gd.data(), dp->d - 1, dp->af[q].p,
                             dp->afT[q].p, dp->rows(q), 1.0, 0.0, st));
  }
  return TSG_OK;
}

int tsg_dplan_solve(tsg_dplan* dp, void* stream) {
  if (!dp) return TSG_EINVAL;
  tsg_ctx* ctx = dp->ctx;
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = pick(dp, stream);
  tsg_plan* pl = dp->pl;
  if (!dp->emulate)
    for (int q = 0; q < dp->nranks; ++q)
      if (q != dp->rank && !dp->peer_x[q])
        return fail(ctx, TSG_EINVAL, "dplan: peers not imported (tsg_dplan_ipc_import)");
  tsg::SolveArgs a{};
  tsg_impl::fill_solve_args(pl, dp->xs[dp->emulate ? 0 : dp->rank].p, a);
  a.nslab = dp->nranks;
  a.sys = dp->emulate ? 0 : 1;
  for (int q = 0; q <= dp->nranks; ++q) a.slo[q] = dp->slo[q];
  for (int q = 0; q < dp->nranks; ++q) {
    double* base = dp->owns(q) ? dp->xs[q].p : dp->peer_x[q];
    a.xs[q] = vbase(base, dp->slo[q], dp->plane);
    a.fs[q] = (dp->emulate || q == dp->rank) ? pl->flags : dp->peer_f[q];
  }
  a.flags = pl->flags;
  a.order = dp->order_own;
  a.ocoord = dp->ocoord_own;
  a.ntiles = dp->ntiles_own;
  a.counter = pl->counter;
  a.status = pl->counter + 1;
  a.epoch = ++dp->epoch;
  TSG_CU(cudaMemsetAsync(pl->counter, 0, sizeof(int), st));
  TSG_CU(cudaMemsetAsync(pl->counter + 1, 0x7f, sizeof(int), st));
  TSG_CU(tsg_impl::launch_plan_solve(pl, a, st));
  return TSG_OK;
}

int tsg_dplan_back_local(tsg_dplan* dp, void* stream) {
  if (!dp) return TSG_EINVAL;
  tsg_ctx* ctx = dp->ctx;
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = pick(dp, stream);
  const int d = dp->d;
  for (int q = 0; q < dp->nranks; ++q) {
    if (!dp->owns(q)) continue;
    const std::vector<int> sd = dp->slab_dims(q);
    const double* src = dp->xs[q].p;
    double* dst_final = dp->emulate ? dp->gath.p + static_cast<int64_t>(q) * dp->rmax * dp->plane : dp->send.p;
    for (int m = 0; m < d - 1; ++m) {
      double* dst = ((d - 2 - m) % 2 == 0) ? dst_final : dp->tmp.p;
      TSG_CU(tsg::mode_product(src, dst, d, sd.data(), m, dp->bwd[m].p, dp->bwdT[m].p, sd[m], 1.0, 0.0, st));
      src = dst;
    }
  }
  return TSG_OK;
}

int tsg_dplan_back_split(tsg_dplan* dp, double* X, void* stream) {
  if (!dp || !X) return TSG_EINVAL;
  tsg_ctx* ctx = dp->ctx;
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = pick(dp, stream);
  std::vector<int> gd = dp->dims;
  gd[dp->d - 1] = dp->nranks * dp->rmax;
  for (int q = 0; q < dp->nranks; ++q) {
    if (!dp->owns(q)) continue;
    double* dst = dp->emulate ? X + static_cast<int64_t>(dp->slo[q]) * dp->plane : X;
    TSG_CU(tsg::mode_product(dp->gath.p, dst, dp->d, gd.data(), dp->d - 1, dp->ab[q].p, dp->abT[q].p,
                             dp->rows(q), 1.0, 0.0, st));
  }
  return TSG_OK;
}

int tsg_dplan_status(tsg_dplan* dp, void* stream) {
  if (!dp) return TSG_EINVAL;
  tsg_ctx* ctx = dp->ctx;
  TSG_CU(cudaSetDevice(ctx->device));
  cudaStream_t st = pick(dp, stream);
  int h[2] = {0, 0};
  TSG_CU(cudaMemcpyAsync(h, dp->pl->counter, sizeof(h), cudaMemcpyDeviceToHost, st));
  TSG_CU(cudaStreamSynchronize(st));
  if (h[1] != 0x7f7f7f7f)
    return fail(ctx, TSG_ESINGULAR, "sharded solve: numerically singular base cell in tile " + std::to_string(h[1]));
  return TSG_OK;
}

}  // extern "C"
