/* tsylv_gpu.h — C-ABI of the B200-native Schur-basis solve.
 *
 * This is the drop-in boundary below the reference's C++ solver entry points
 * (proj/include/tsylv/ headers).  No C++ or torch types cross it: plain
 * pointers, int extents, column-major FP64 buffers (mode 0 fastest, the
 * layout of tsylv::Tensor, tensor.hpp:19-27).  Each entry point names the
 * reference interface it replaces.
 *
 * Status codes (mirror tools/tsylv.cpp:1-5 exit codes; the C++ shim in
 * include/tsylv/ rethrows the reference exception types, errors.hpp:13-62):
 *   TSG_OK 0, TSG_EDIM 1 (dimension_error), TSG_ESINGULAR 2 (singular_error),
 *   TSG_EFACT 3 (factorization_error), TSG_EINVAL 4 (std::invalid_argument),
 *   TSG_ECUDA 5 (CUDA/NCCL failure -> std::runtime_error).
 *
 * Ownership: the caller owns every host buffer; the context owns all device
 * memory.  One context per host thread (not thread-safe); several contexts
 * may coexist.  Calls are synchronous unless opts->stream is set.
 */
#ifndef TSYLV_GPU_H
#define TSYLV_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSG_OK 0
#define TSG_EDIM 1
#define TSG_ESINGULAR 2
#define TSG_EFACT 3
#define TSG_EINVAL 4
#define TSG_ECUDA 5

#define TSG_MAX_ORDER 8

typedef struct tsg_ctx tsg_ctx;
typedef struct tsg_plan tsg_plan;

typedef struct {
  int n_min;             /* base-tile extent bound per mode (0 = tuned default) */
  int tile[TSG_MAX_ORDER]; /* explicit per-mode tile extents (0 = from n_min) */
  int inputs_on_device;  /* 1: B/X are device pointers (resident in HBM) */
  void* stream;          /* cudaStream_t to run on (NULL = context stream) */
  /* plans only: modes whose transforms are the identity (bit m), their U may
   * be NULL; and the free mode of the eigen-decoupled solve (-1: chosen by
   * the plan).  The slab-sharded decoupled solve (paper_1905_09539_b200/dist.py)
   * runs a plan's transforms and its fibre solve on different slabs. */
  int skip_transform_mask;
  int free_mode;
} tsg_opts;

typedef struct {
  double t_fwd_ms;       /* forward transforms (B ->B~), CUDA events */
  double t_solve_ms;     /* reduced (quasi-)triangular solve */
  double t_back_ms;      /* back transforms (X~ -> X) */
  double t_h2d_ms;       /* host->device copy (host inputs only) */
  double t_d2h_ms;       /* device->host copy (host inputs only) */
  double t_total_ms;     /* whole execute(), CUDA events */
  double flops_alg;      /* algorithmic FLOP credited */
  double flops_exec;     /* FLOP actually issued by the schedule */
  int zero_pivot_index;  /* -1, or first linear index of a singular base cell */
  int kernel_launches;   /* kernels launched by execute() */
} tsg_report;

void tsg_default_opts(tsg_opts* o);

/* Context: device, streams, workspace. */
int tsg_create(int n_gpus, const int* device_ids, tsg_ctx** out);
void tsg_destroy(tsg_ctx* ctx);
const char* tsg_last_error(const tsg_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) — lets callers time execute()
 * with CUDA events on the stream the kernels are launched on. */
void* tsg_ctx_stream(const tsg_ctx* ctx);

/* ---- Laplace-like: sum_m X x_m A_m = B  (laplace.hpp:248-302) ----------
 * Real Schur basis A_m = U_m T_m U_m^T: T[m] upper quasi-triangular,
 * U[m] orthogonal, both dims[m] x dims[m] column-major host arrays.
 * Replaces laplace.hpp:276-298 (forward transforms, reduced solve, back
 * transforms).  X may alias B. */
int tsg_laplace_solve(tsg_ctx* ctx, int d, const int* dims,
                      const double* const* T, const double* const* U,
                      const double* B, double* X, const tsg_opts* opts,
                      tsg_report* rep);

/* Reduced form only (laplace_recursive, laplace.hpp:185-195): solves
 * sum_m Xt x_m T_m = Bt for quasi-triangular T_m. */
int tsg_laplace_reduced(tsg_ctx* ctx, int d, const int* dims,
                        const double* const* T, const double* Bt, double* Xt,
                        const tsg_opts* opts, tsg_report* rep);

/* ---- Generalized: X x_0 A_0 + X x_0 C x_1 A_1 ... = B  (gsylv.hpp:236-302)
 * qz(A_0, C) = (Q, Z, S, Tc): A_0 = Q S Z^T, C = Q Tc Z^T; tail m >= 1:
 * A_m = U_m T_m U_m^T.  Ttail/Utail hold d-1 pointers (modes 1..d-1). */
int tsg_gsylv_solve(tsg_ctx* ctx, int d, const int* dims, const double* S,
                    const double* Tc, const double* Q, const double* Z,
                    const double* const* Ttail, const double* const* Utail,
                    const double* B, double* X, const tsg_opts* opts,
                    tsg_report* rep);

/* Reduced form only (gsylv_recursive, gsylv.hpp:149-159). */
int tsg_gsylv_reduced(tsg_ctx* ctx, int d, const int* dims, const double* S,
                      const double* Tc, const double* const* Ttail,
                      const double* Bt, double* Xt, const tsg_opts* opts,
                      tsg_report* rep);

/* ---- Plans: set up once (factors uploaded, tiles/schedule built), execute
 * many times.  The bench times tsg_plan_enqueue with inputs resident.
 * family: 0 Laplace (Tc/S/Q/Z unused), 1 gsylv.  For gsylv, T[0]=S,
 * U[0]=Q and the extra pointers Tc, Z are used.  reduced_only=1 skips
 * both transforms (U/Q/Z may be NULL). */
int tsg_plan_create(tsg_ctx* ctx, int family, int d, const int* dims,
                    const double* const* T, const double* const* U,
                    const double* Tc, const double* Z, int reduced_only,
                    const tsg_opts* opts, tsg_plan** out);
int tsg_plan_execute(tsg_plan* plan, const double* B, double* X,
                     int inputs_on_device, tsg_report* rep);
/* Asynchronous device-resident solve: enqueue the whole pipeline for B -> X
 * (device pointers) on the context stream and return at once, so repeated
 * solves run back to back without host round trips.  No singularity check
 * and no timings: tsg_plan_sync waits for every enqueued solve and reports
 * the zero pivot of the most recent one (rep may be NULL). */
int tsg_plan_enqueue(tsg_plan* plan, const double* B, double* X);
int tsg_plan_sync(tsg_plan* plan, tsg_report* rep);
/* serial = 1: launch every kernel of a solve after its predecessor (no
 * overlap of the back transform with the solve's drain, no trailing-cube
 * grid), so the per-phase times of tsg_plan_execute are per-kernel times.
 * Default 0.  Same results either way (bit-identical). */
int tsg_plan_set_serial(tsg_plan* plan, int serial);
/* Transforms only (dir 0: forward B x_m U_m^T, 1: back X x_m U_m; the
 * decoupled plan's folded eigenbasis transforms), in -> out (distinct device
 * buffers), on `stream` (NULL = context stream). */
int tsg_plan_transform(tsg_plan* plan, int dir, const double* in, double* out, void* stream);
/* Eigen-decoupled plans: the free mode (-1 if the plan is not decoupled). */
int tsg_plan_free_mode(const tsg_plan* plan);
void tsg_plan_destroy(tsg_plan* plan);
/* Solve nrhs right-hand sides from HOST buffers B[i] into X[i] (pinned
 * memory recommended) with the copies overlapped: the host->device copy of
 * B[i+1] and the device->host copy of X[i-1] run on copy streams while
 * solve i runs (two device staging slots).  Synchronous on return;
 * rep->t_total_ms covers the whole batch (first copy to last copy). */
int tsg_plan_execute_stream(tsg_plan* plan, int nrhs, const double* const* B, double* const* X,
                            tsg_report* rep);
/* Number of tiles / dataflow steps of the plan's reduced solve. */
int tsg_plan_info(const tsg_plan* plan, int64_t* n_tiles, int* tile_extents,
                  double* flops_alg);

/* Which reduced-solve kernel the plan runs, as a short text
 * ("decoupled f=<mode> kappa=<prod>", "lap16", "lap3", "lapd", "gsyd",
 * "generic"); returns the string length (truncated to len - 1). */
int tsg_plan_describe(const tsg_plan* plan, char* buf, int len);

/* ---- Mode product Y = X x_mode A  (tensor.hpp:187-231) -----------------
 * A is r x dims[mode] column-major; Y has dims with dims[mode] -> r. */
int tsg_mode_multiply(tsg_ctx* ctx, int d, const int* dims, const double* X,
                      int r, const double* A, int mode, double* Y,
                      const tsg_opts* opts);

/* ---- Relative residual (oracle.hpp:231-268) on the device -------------
 * ||op(X) - B||_F / (scale ||X||_F + ||B||_F) with scale = sum_m ||A_m||_F
 * (Laplace, family 0) or ||A_0||_F + ||C||_F prod_{m>=1} ||A_m||_F (gsylv,
 * family 1), computed through mode products only.  A holds the d dense
 * ORIGINAL coefficients; C is NULL for Laplace.  B/X follow inputs_on_device. */
/* Solvability screen on the GPU (reference solvability.hpp:31-116): the
 * smallest |operator eigenvalue| over every eigenvalue tuple of the
 * quasi-triangular factors, its first position in the reference's scan order
 * (witness: Laplace one index per mode; gsylv the 2x2/1x1 block's first row of
 * S, then one index per tail mode), solvable = min_abs > tol (tol <= 0:
 * unit roundoff times the sum of the factors' Frobenius norms). */
int tsg_screen_laplace(tsg_ctx* ctx, int d, const int* dims, const double* const* T, double tol,
                       double* min_abs, int* witness, int* solvable);
int tsg_screen_gsylv(tsg_ctx* ctx, int d, const int* dims, const double* S, const double* Tc,
                     const double* const* Ttail, double tol, double* min_abs, int* witness, int* solvable);
int tsg_residual(tsg_ctx* ctx, int family, int d, const int* dims,
                 const double* const* A, const double* C, const double* B,
                 const double* X, int inputs_on_device, double* out);

/* ---- Complex scalars (T = std::complex<double>) -----
 * Same entry points for complex problems: every matrix and tensor buffer is
 * interleaved (re, im) FP64, the layout of std::complex<double> arrays.
 * Factors come from the complex Schur / QZ decompositions (zgees / zgges):
 * T, S, Tc upper triangular, U, Q, Z unitary; forward transforms use the
 * adjoints (laplace.hpp:282, gsylv.hpp:278-280).  Replace the T = Complex
 * instantiations of laplace.hpp:276-298, gsylv.hpp:272-298 (solve),
 * laplace.hpp:185-195 / gsylv.hpp:149-159 (reduced), tensor.hpp:187-231
 * (mode product) and oracle.hpp:233-268 (residual).  opts->free_mode picks
 * the Laplace free mode of the eigen-decoupled solve (-1 = automatic). */
int tsg_zlaplace_solve(tsg_ctx* ctx, int d, const int* dims, const double* const* T,
                       const double* const* U, const double* B, double* X,
                       const tsg_opts* opts, tsg_report* rep);
int tsg_zlaplace_reduced(tsg_ctx* ctx, int d, const int* dims, const double* const* T,
                         const double* Bt, double* Xt, const tsg_opts* opts, tsg_report* rep);
int tsg_zgsylv_solve(tsg_ctx* ctx, int d, const int* dims, const double* S, const double* Tc,
                     const double* Q, const double* Z, const double* const* Ttail,
                     const double* const* Utail, const double* B, double* X,
                     const tsg_opts* opts, tsg_report* rep);
int tsg_zgsylv_reduced(tsg_ctx* ctx, int d, const int* dims, const double* S, const double* Tc,
                       const double* const* Ttail, const double* Bt, double* Xt,
                       const tsg_opts* opts, tsg_report* rep);
int tsg_zmode_multiply(tsg_ctx* ctx, int d, const int* dims, const double* X, int r,
                       const double* A, int mode, double* Y, const tsg_opts* opts);
int tsg_zresidual(tsg_ctx* ctx, int family, int d, const int* dims, const double* const* A,
                  const double* C, const double* B, const double* X, int inputs_on_device,
                  double* out);

/* ABI version (bumped on any signature change). */

/* ---- Slab-sharded multi-GPU solve (Laplace-like, d = 3) ---------------------
 * Replaces nothing in the reference (a CPU library); implements the
 * multi-GPU plan of SURVEY.md §8(e) behind the same algorithm as
 * tsg_laplace_solve.  The tensor is cut into `nranks` slabs along its LAST
 * mode (tile-aligned, never inside a 2x2 Schur block; a slab is a contiguous
 * piece of the column-major tensor).  One process per GPU owns one slab:
 *   forward_local   B_r x_m U_m^T, m < d-1          -> send buffer (padded)
 *   (caller)        all-gather of the send buffers   -> gather buffer (NCCL)
 *   forward_split   gather x_{d-1} U_{d-1}^T[R_r,:]  -> own slab of B~
 *   solve           one dataflow kernel per GPU over all slabs: tiles and
 *                   flags of the other ranks are read through CUDA IPC peer
 *                   mappings over NVLink (system-scope acquire/release)
 *   back_local / (caller) all-gather / back_split    -> X_r
 * Emulated mode (emulate = 1): one process holds all slabs on one GPU, the
 * gather buffer doubles as the send buffers and `solve` runs one kernel over
 * every slab (validates the sharded path on a single device); B and X are
 * then the whole tensor.  Every step is enqueued on `stream` (cudaStream_t,
 * NULL = context stream) without host synchronisation. */
typedef struct tsg_dplan tsg_dplan;
#define TSG_IPC_BYTES 128
/* Slab row bounds (nranks + 1 entries) of a mode of extent n with
 * quasi-triangular factor T, for base tiles of extent `tile`. */
int tsg_slab_bounds(int n, const double* T, int tile, int nranks, int* bounds);
/* Re-sharding pack (dir 0) / unpack (dir 1) of the decoupled sharded solve on
 * the device: `rows` contiguous runs of n0 doubles <-> nranks segments, segment
 * q = columns [b0[q], b0[q+1]) of every run, (rows, w_q) row-major at offset
 * rows * b0[q] (the send layout of the all-to-all; b0: nranks + 1 host ints,
 * nranks <= 64).  src and dst are device buffers of rows * n0 doubles. */
int tsg_slab_pack(tsg_ctx* ctx, const double* src, double* dst, long long rows, int n0, int nranks,
                  const int* b0, int dir, void* stream);
int tsg_dplan_create(tsg_ctx* ctx, int rank, int nranks, int emulate, int d, const int* dims,
                     const double* const* T, const double* const* U, const tsg_opts* opts,
                     tsg_dplan** out);
void tsg_dplan_destroy(tsg_dplan* dp);
/* slab bounds (nranks + 1), elements of this rank's slab, of one send slot */
int tsg_dplan_info(const tsg_dplan* dp, int* bounds, int64_t* slab_elems, int64_t* send_elems);
int tsg_dplan_buffers(tsg_dplan* dp, double** send, double** gather);
int tsg_dplan_ipc_export(tsg_dplan* dp, void* handles);
int tsg_dplan_ipc_import(tsg_dplan* dp, const void* all_handles);
int tsg_dplan_forward_local(tsg_dplan* dp, const double* B, void* stream);
int tsg_dplan_forward_split(tsg_dplan* dp, void* stream);
int tsg_dplan_solve(tsg_dplan* dp, void* stream);
int tsg_dplan_back_local(tsg_dplan* dp, void* stream);
int tsg_dplan_back_split(tsg_dplan* dp, double* X, void* stream);
/* Synchronises the stream; TSG_ESINGULAR when a zero pivot was seen. */
int tsg_dplan_status(tsg_dplan* dp, void* stream);

int tsg_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TSYLV_GPU_H */
