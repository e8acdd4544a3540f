"""Benchmark of the B200 Schur-basis solve (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Headline workload: C4 (Laplace d=3, 1024x512x256), the configuration
BASELINE.json quotes the 1/2/4/8-GPU metric on.  One "step" is one full solve
of that configuration — forward
transforms B~ = B x_m U_m^T, the reduced quasi-triangular dataflow solve,
back transforms X = X~ x_m U_m — on synthetic seeded inputs
(include/tsylv/random.hpp).  The Schur/QZ factors are shared host setup
(BASELINE.json north_star) and are computed once, outside the timed region.

  value : unknowns/s of the whole job with B resident in HBM (device-timed,
          CUDA events on the library's stream, max over ranks)
  e2e   : the same metric through the C-ABI with HOST buffers (pinned),
          H2D + D2H of every step inside the timed region
          (tsg_plan_execute_stream overlaps them with the neighbouring solves)
  roofline : dominant kernel's algorithmic FLOP / its average launch time,
          against the measured FP64 DMMA peak (profiles/r01_fp64_peak_probe.log)
  cpu_baseline : the reference solver itself (oracle/_ref, built from the
          unmodified reference headers) on the host cores, rank 0 at N=1;
          its solution also gives `rel_err_vs_reference` of the timed output
  all_configs : C1-C5 (one plan each, K solves enqueued back to back):
          ms per solve, unknowns/s, fraction of the FP64 peak, residual

Multi-GPU (N>1, torchrun, NCCL): the Laplace configurations (C1-C4) run ONE
problem sharded over the N GPUs (strong scaling), eigen-decoupled: each rank
holds a slab along the last mode; the transforms of modes 0..d-2 run there,
two NCCL all-to-alls per solve move the data to slabs along mode 0 and back,
where the last mode's transforms and the fibre solve along the free mode run
(paper_1905_09539_b200/dist.py, DecoupledSharded).  `--sharded-ipc` runs the
tile-DAG path over peer-mapped slabs instead (d = 3).  C5 (gsylv) runs one
replica per GPU (weak scaling).  `--sharded` forces the sharded path at N=1
(plumbing check).  `--impl reference` times the reference CPU solver (rank 0
only; other ranks exit 0) on inputs drawn from the reference's own
RandomStream (oracle/_ref), so that process never loads the product library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs (kind: 1 convection-diffusion Laplace, 2 G/sqrt(n)+3I
# Laplace, 5 gsylv posed as coeffs {A, C^T, C^T, C^T}, c = B).
CONFIGS = {
    "C1": (1, (64, 64, 64), "Laplace d=3 64^3 convection-diffusion"),
    "C2": (2, (256, 256, 256), "Laplace d=3 256^3, A_mu = G/sqrt(n)+3I"),
    "C3": (2, (24,) * 6, "Laplace d=6 24^6, A_mu = G/sqrt(24)+3I"),
    "C4": (2, (1024, 512, 256), "Laplace d=3 1024x512x256, A_mu = G/sqrt(n)+3I"),
    "C5": (5, (200, 40, 40, 40), "gsylv A X + B X (C(x)C(x)C) = D, 200x64000"),
}
PEAK_FP64_TFLOPS = 37.07  # measured DMMA peak, profiles/r01_fp64_peak_probe.log
METRIC = "FP64 Schur-basis solve throughput"
UNIT = "unknowns/s"


def flops_alg(kind: int, dims) -> tuple[float, float]:
    """(transform FLOP, solve FLOP) credited per solve."""
    N = float(np.prod(dims))
    sn = float(sum(dims))
    tr = 4.0 * N * sn
    if kind == 5:
        solve = N * ((dims[0] - 1) + (dims[0] + sum(dims[1:])))
    else:
        solve = N * sum(n - 1 for n in dims)
    return tr, solve


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_of(name: str) -> dict:
    """The `config` object both arms print (identical keys and values)."""
    kind, dims, desc = CONFIGS[name]
    return {"workload": name, "desc": desc, "dims": list(dims), "unknowns": int(np.prod(dims)),
            "seed": 1}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_plan(T, ctx, kind, p):
    from paper_1905_09539_b200.plan import Plan
    if kind == 5:
        q, z, s, tc = T.qz(p.coeffs[0], p.c)
        fs = [T.schur(a) for a in p.coeffs[1:]]
        return Plan(ctx, 1, [s] + [f[1] for f in fs], [q] + [f[0] for f in fs], Tc=tc, Z=z)
    fs = [T.schur(a) for a in p.coeffs]
    return Plan(ctx, 0, [f[1] for f in fs], [f[0] for f in fs])


def traffic_from_profiles(config: str, kernel: str):
    """ncu dram bytes (read + write) per launch of `kernel` ("solve" or
    "dgemm"), if an ncu --set full capture of this config was summarised into
    profiles/ncu_traffic.json (tools/ncu_summary.py)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f).get(config)
    except (OSError, ValueError):
        return None
    if isinstance(d, dict):
        return d.get(kernel)
    return d if kernel == "solve" else None


def cpu_reference_solve(kind, dims, seed=1, problem=None):
    """One reference solve (oracle/_ref) on the box's host cores, on the
    BASELINE inputs drawn from the reference's own RandomStream (or on
    `problem` = (coeffs, c, rhs)).  Returns (seconds like-for-like, seconds
    total, info, cores, X, reference config name)."""
    cores = os.cpu_count() or 1
    os.environ["OPENBLAS_NUM_THREADS"] = str(cores)
    os.environ.pop("TSYLV_THREADS", None)
    import oracle.ref as R
    co, c, rhs = problem if problem is not None else R.baseline_problem(kind, dims, seed=seed)
    t0 = time.perf_counter()
    if kind == 5:
        # the reference's own default (merge + complex); real recursion takes minutes at C5
        x, info = R.solve_gsylv(co, c, rhs, strategy=1, arithmetic=0)
        name = "merge+complex_triangular (reference default)"
    elif len(dims) > 3:
        # C3: real recursion exceeds 5 min (3^6 base blocks); the default is ~2 min
        x, info = R.solve_laplace(co, rhs, strategy=1, arithmetic=0)
        name = "merge+complex_triangular (reference default)"
    else:
        x, info = R.solve_laplace(co, rhs, strategy=0, arithmetic=1)
        name = "recursion_only+real_quasitriangular (the GPU path's arithmetic)"
    total = time.perf_counter() - t0
    like = info[3] + info[4]  # recursion_s + back_transform_s (Schur excluded)
    return like, total, info, cores, x, name


def run_reference(a, rank):
    """The reference arm: the reference's own CPU solver (oracle/_ref) on all
    host cores, rank 0 only.  Each step is one full solve of the workload
    (about 1.5 min at C4 on 16 cores), so the run stops after --steps solves
    or once 150 s of solves have run (at least one), with no warm-up (plain
    CPU code: nothing to warm); the cap is stated in the line."""
    if rank != 0:
        return
    kind, dims, desc = CONFIGS[a.config]
    N = float(np.prod(dims))
    vals, tots = [], []
    t_start = time.perf_counter()
    while len(vals) < max(a.steps, 1) and (not vals or time.perf_counter() - t_start < 150.0):
        like, total, info, cores, x, cfg_name = cpu_reference_solve(kind, dims)
        del x
        vals.append(like)
        tots.append(total)
    steps = len(vals)
    t = min(vals)
    v = N / t
    sample = (f"{steps} full {a.config} solve(s) of the reference tsylv ({cfg_name}; oracle/_ref, "
              f"unmodified headers + OpenBLAS 0.3.15, OPENBLAS_NUM_THREADS={cores}); value = N / "
              f"min(recursion_s + back_transform_s), Schur setup excluded; total incl. Schur "
              f"{min(tots):.2f} s")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
        "steps": steps, "warmup": 0, "ms_per_step": t * 1e3,
        "steps_note": f"requested --steps {a.steps} --warmup {a.warmup}; ran {steps} timed solve(s) "
                      f"and no warm-up (150 s budget; one step is one full CPU solve, "
                      f"{t:.2f} s like-for-like)",
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded RandomStream, BASELINE.json distributions)",
        "config": config_of(a.config),
        "reference_config": cfg_name,
        "cpu": {"model": cpu_model(), "cores": cores},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def time_enqueued(torch, plan, stream, b, x, steps):
    """K solves enqueued back to back on the library stream (tsg_plan_enqueue,
    no host round trip between steps), CUDA events on that stream.
    Returns (ms per solve, kernel launches per solve)."""
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
    for _ in range(steps):
        plan.enqueue_device(b.data_ptr(), x.data_ptr())
    with torch.cuda.stream(stream):
        e1.record(stream)
    e1.synchronize()
    rep = plan.sync()
    if rep.zero_pivot_index >= 0:
        raise RuntimeError(f"singular operator (zero pivot {rep.zero_pivot_index})")
    return e0.elapsed_time(e1) / steps, rep.kernel_launches


def all_configs(T, torch, ctx, local, steps, skip):
    """C1-C5 on this GPU: one plan each, K solves enqueued back to back."""
    out = {}
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", local))
    for name in CONFIGS:
        if name == skip:
            continue
        kind, dims, _ = CONFIGS[name]
        N = int(np.prod(dims))
        p = T.make_problem(kind, dims, seed=1)
        plan = build_plan(T, ctx, kind, p)
        b = torch.from_numpy(np.ascontiguousarray(p.rhs.reshape(-1, order="F"))).cuda(local)
        x = torch.empty_like(b)
        for _ in range(3):
            plan.execute_device(b.data_ptr(), x.data_ptr())
        torch.cuda.synchronize()
        ms, launches = time_enqueued(torch, plan, stream, b, x, steps)
        res = T.residual(p, x.cpu().numpy().reshape(dims, order="F"))
        tr_f, solve_f = flops_alg(kind, dims)
        out[name] = {"ms_per_solve": ms, "reduced_solve": plan.describe(), "unknowns_per_s": N / (ms * 1e-3),
                     "fp64_tflops_alg": (tr_f + solve_f) / (ms * 1e-3) / 1e12,
                     "frac_fp64_peak_alg": (tr_f + solve_f) / (ms * 1e-3) / 1e12 / PEAK_FP64_TFLOPS,
                     "residual": res, "solves": steps, "launches_per_solve": launches}
        plan.close()
        del b, x, p
        torch.cuda.empty_cache()
    return out


# Complex-scalar workloads: the reference's dense
# complex generators (random_laplace_problem / random_gsylv_problem with
# T = Complex, seed 1) at the C2 / C5 shapes.
COMPLEX_CONFIGS = {"Z2": ("laplace", (256, 256, 256)), "Z5": ("gsylv", (200, 40, 40, 40))}


def complex_configs(T, reps=3):
    """Complex solves through the drop-in API (solve_laplace<Complex> /
    solve_gsylv<Complex>: host zgees/zgges, then the GPU); the device phases
    (forward + reduced solve + back, CUDA events) are the figure, best of
    `reps` after one warm-up; h2d/d2h and the host Schur are reported apart."""
    out = {}
    for name, (fam, dims) in COMPLEX_CONFIGS.items():
        p = T.random_problem(fam, dims, seed=1)
        solve = T.solve_laplace if fam == "laplace" else T.solve_gsylv
        solve(p)
        best = None
        for _ in range(reps):
            rep = solve(p)
            g = rep.gpu
            dev = g["fwd_ms"] + g["solve_ms"] + g["back_ms"]
            if best is None or dev < best[0]:
                best = (dev, rep)
        dev, rep = best
        g = rep.gpu
        N = int(np.prod(dims))
        out[name] = {"family": fam, "dims": list(dims), "scalar": "complex128",
                     "device_ms_per_solve": dev, "fwd_ms": g["fwd_ms"], "solve_ms": g["solve_ms"],
                     "back_ms": g["back_ms"], "h2d_ms": g["h2d_ms"], "d2h_ms": g["d2h_ms"],
                     "unknowns_per_s": N / (dev * 1e-3),
                     "fp64_tflops_alg": g["flops_alg"] / (dev * 1e-3) / 1e12,
                     "frac_fp64_peak_alg": g["flops_alg"] / (dev * 1e-3) / 1e12 / PEAK_FP64_TFLOPS,
                     "residual": rep.residual, "host_schur_s": rep.timings.reduction_s}
        del p, rep
    return out


def run_ours(a, rank, world, local):
    import torch
    import paper_1905_09539_b200 as T
    from paper_1905_09539_b200.plan import Context

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    kind, dims, desc = CONFIGS[a.config]
    N = int(np.prod(dims))
    p = T.make_problem(kind, dims, seed=1 + rank)
    ctx = Context(local)
    plan = build_plan(T, ctx, kind, p)
    info = plan.info()
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", local))
    b_host = torch.from_numpy(np.ascontiguousarray(p.rhs.reshape(-1, order="F"))).pin_memory()
    x_host = torch.empty_like(b_host).pin_memory()
    b = b_host.cuda()
    x = torch.empty_like(b)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (device-resident and host-buffer paths)
    for _ in range(max(a.warmup, 3)):
        plan.execute_device(b.data_ptr(), x.data_ptr())
    plan.execute_host(b_host.numpy(), x_host.numpy())

    # per-phase split (CUDA events inside each solve; outside the timed region)
    reps = [plan.execute_device(b.data_ptr(), x.data_ptr()) for _ in range(3)]

    # ---- device-resident timed region --------------------------------------
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    time.sleep(0.2)
    ms, launches_per = time_enqueued(torch, plan, stream, b, x, a.steps)
    clk = clocks.stop()
    barrier()
    launches = a.steps * launches_per

    # ---- end-to-end through the C-ABI with host buffers -----------------------
    # tsg_plan_execute_stream: every step copies its right-hand side from
    # pinned host memory and its solution back; the copies of step i+1 / i-1
    # overlap the solve of step i (two device staging slots).  Timed by CUDA
    # events from the first host->device copy to the last device->host copy.
    plan.execute_stream([b_host.data_ptr()] * 2, [x_host.data_ptr()] * 2)  # warm-up
    barrier()
    srep = plan.execute_stream([b_host.data_ptr()] * a.steps, [x_host.data_ptr()] * a.steps)
    barrier()
    ms_e2e = srep.t_total_ms / a.steps

    # max over ranks
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms, ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e = float(t[0]), float(t[1])

    # correctness of the timed output (device residual through mode products)
    xs = x.cpu().numpy().reshape(dims, order="F")
    res = T.residual(p, xs)

    tr_f, solve_f = flops_alg(kind, dims)
    t_fwd = statistics.median(r.t_fwd_ms for r in reps)
    t_solve_ovl = statistics.median(r.t_solve_ms for r in reps)
    t_back_rest = statistics.median(r.t_back_ms for r in reps)
    # Kernel-timing leg (outside the timed region): in the timed steps the
    # back transform's mode-0 GEMM overlaps the solve's drain (tile-flag gate,
    # programmatic launch), so the solve kernel's own launch time is taken
    # from a few steps with the gate off (TSG_GATE=0 -> back after solve).
    plan.set_serial(True)
    try:
        kreps = [plan.execute_device(b.data_ptr(), x.data_ptr()) for _ in range(5)]
    finally:
        plan.set_serial(False)
    t_solve = statistics.median(r.t_solve_ms for r in kreps)
    t_back = statistics.median(r.t_back_ms for r in kreps)
    t_fwd_k = statistics.median(r.t_fwd_ms for r in kreps)
    # dominant kernel (by its share of the step, from the kernel-timing leg
    # where every kernel runs alone): the dataflow solve (1 launch) vs the
    # DMMA transform GEMM (2d launches); achieved = algorithmic FLOP per
    # launch / launch time
    t_fwd_gated, t_fwd = t_fwd, t_fwd_k
    d = len(dims)
    if t_solve >= t_fwd + t_back:
        dom = {"kernel": "solve kernel (reduced dataflow solve, K2+K3)", "ncu": "solve",
               "achieved": solve_f / (t_solve * 1e-3) / 1e12, "launch_ms": t_solve}
    else:
        dom = {"kernel": "dgemm_tma_kernel (mode transforms, K1: TMA-staged DMMA GEMM)", "ncu": "dgemm",
               "achieved": tr_f / ((t_fwd + t_back) * 1e-3) / 1e12,
               "launch_ms": (t_fwd + t_back) / (2 * d)}
    traffic = traffic_from_profiles(a.config, dom["ncu"])
    roofline = {"bound": "tensor", "achieved": dom["achieved"], "peak": PEAK_FP64_TFLOPS,
                "unit": "TFLOP/s", "frac": dom["achieved"] / PEAK_FP64_TFLOPS,
                "traffic": traffic, "kernel": dom["kernel"],
                "peak_source": "measured FP64 DMMA peak (mma.sync m8n8k4 f64 loop, "
                               "profiles/r01_fp64_peak_probe.log); MEASURED_PEAKS.json has no FP64 entry"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": world * N / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": max(a.warmup, 3), "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "weak" if world > 1 else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded RandomStream, BASELINE.json distributions)",
            "config": config_of(a.config),
            "details": {
                "l2": "inputs larger than L2 (8N bytes per tensor, plus two N-sized work "
                      "buffers, > 126 MB L2)",
                "parallelism": (f"{world} independent replicas (sharded setup failed: "
                                f"{getattr(a, 'fallback', '')})" if getattr(a, "fallback", None)
                                else f"{world} independent replicas (no sharding)") if world > 1
                else "single GPU", "tiles": info["n_tiles"], "tile": info["tile"],
                "reduced_solve": plan.describe(),
                "schur_setup": "host LAPACK dgees/dgges, outside the timed region"},
            "phases_ms": {"forward_transforms_before_solve": t_fwd_gated,
                          "last_fwd_gemm+solve+back_modes_overlapped": t_solve_ovl,
                          "back_transforms_rest": t_back_rest,
                          "alone_forward_transforms": t_fwd, "alone_reduced_solve": t_solve,
                          "alone_back_transforms": t_back},
            "fp64_tflops_alg": (tr_f + solve_f) / (ms * 1e-3) / 1e12,
            "frac_fp64_peak_alg": (tr_f + solve_f) / (ms * 1e-3) / 1e12 / PEAK_FP64_TFLOPS,
            "residual": res,
            "roofline": roofline,
            "e2e": {"value": world * N / (ms_e2e * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N,
                    "ms_per_step": ms_e2e,
                    "api": "tsg_plan_execute_stream (pinned host buffers, copies overlapped with "
                           "the neighbouring steps' solves)"},
            "gpu_launches": launches,
            "clocks": clk,
        }
        if world == 1 and not a.no_all_configs:
            plan.close()
            del b, x
            torch.cuda.empty_cache()
            line["all_configs"] = all_configs(T, torch, ctx, local, 10, a.config)
            line["complex_configs"] = complex_configs(T)
        if world == 1 and not a.no_cpu_baseline:
            like, total, rinfo, cores, xr, cfg_name = cpu_reference_solve(
                kind, dims, problem=(p.coeffs, getattr(p, "c", None), p.rhs))
            nr = float(np.linalg.norm(xr))
            line["rel_err_vs_reference"] = float(np.linalg.norm(xs - xr) / nr)
            line["reference_residual"] = rinfo[0]
            line["cpu"] = {"model": cpu_model(), "cores": cores}
            line["cpu_baseline"] = {
                "value": N / like, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"one full {a.config} solve of the reference tsylv ({cfg_name}; "
                          f"oracle/_ref, unmodified headers + OpenBLAS, OPENBLAS_NUM_THREADS="
                          f"{cores}) on the same inputs; value = N/(recursion_s+back_transform_s) "
                          f"= N/{like:.2f}s, Schur excluded (total incl. Schur {total:.2f}s); "
                          f"its X gives rel_err_vs_reference"}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_sharded(a, rank, world, local):
    """One problem sharded over `world` GPUs (strong scaling), eigen-decoupled:
    last-mode slabs <-> mode-0 slabs by two NCCL all-to-alls around a local
    fibre solve (paper_1905_09539_b200.dist.DecoupledSharded).
    `--sharded-ipc` runs the tile-DAG path with peer-mapped slabs instead."""
    import torch
    import torch.distributed as dist
    import paper_1905_09539_b200 as T
    from paper_1905_09539_b200.plan import Context

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    kind, dims, desc = CONFIGS[a.config]
    N = int(np.prod(dims))
    p = T.make_problem(kind, dims, seed=1)  # the same problem on every rank
    fs = [T.schur(c) for c in p.coeffs]      # shared host setup
    ctx = Context(local)
    # sharded setup; if it fails on any rank, every rank falls back to one
    # independent replica per GPU (reported in the line)
    err = ""
    mode = "ipc" if a.sharded_ipc else "decoupled"
    try:
        if os.environ.get("TSG_BENCH_SHARD_FAIL"):  # exercise the fallback (development)
            raise RuntimeError("forced by TSG_BENCH_SHARD_FAIL")
        if mode == "decoupled":
            from paper_1905_09539_b200.dist import DecoupledSharded, DeviceDecoupled
            # pipeline chunks per slab: the all-to-alls overlap the phase-A/C transforms
            # of the neighbouring chunks; 1 = one exchange per direction
            nchunk = a.chunks if a.chunks > 0 else (4 if world > 1 else 1)
            nchunk = max(1, min(nchunk, min(dims[-1] // world // 8, 16) or 1))
            be = DeviceDecoupled(ctx, rank, world, [f[1] for f in fs], [f[0] for f in fs], chunks=nchunk)
            sl = DecoupledSharded(be)
        else:
            from paper_1905_09539_b200.dist import DeviceSlabs, ShardedLaplace
            be = DeviceSlabs(ctx, rank, world, [f[1] for f in fs], [f[0] for f in fs])
            sl = ShardedLaplace(be)
    except Exception as e:  # noqa: BLE001
        err = f"{type(e).__name__}: {e}"[:200]
    flag = torch.tensor([1.0 if err else 0.0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX)
    if float(flag) > 0:
        if rank == 0:
            print(f"[bench] sharded setup failed ({err or 'on another rank'}); running replicas",
                  file=sys.stderr, flush=True)
        a.fallback = err or "sharded setup failed on another rank"
        return run_ours(a, rank, world, local)
    bounds = be.bd if mode == "decoupled" else be.bounds
    lo, hi = bounds[rank], bounds[rank + 1]
    b_host = torch.from_numpy(np.ascontiguousarray(p.rhs[..., lo:hi].reshape(-1, order="F"))).pin_memory()
    x_host = torch.empty_like(b_host).pin_memory()
    b = b_host.to(dev)
    x = torch.empty_like(b)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=dev)
    sp = ctx.stream_ptr()

    if mode == "decoupled":
        def step():
            sl.solve(b, x)
    else:
        def step():
            be.forward_local(b, sp)
            sl._all_gather(sp)
            be.forward_split(sp)
            be.solve(sp)
            be.back_local(sp)
            sl._all_gather(sp)
            be.back_split(x, sp)

    with torch.cuda.stream(stream):
        for _ in range(max(a.warmup, 3)):
            step()
        if mode == "decoupled":
            be.check()
        else:
            be.status(sp)
        dist.barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(local)
        clocks.start()
        time.sleep(0.2)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            step()
        e1.record(stream)
        stream.synchronize()
        clk = clocks.stop()
        ms = e0.elapsed_time(e1) / a.steps
        if mode == "decoupled":
            be.check()
        else:
            be.status(sp)
        # end to end: pinned host slab in, solution slab out, every step
        dist.barrier()
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(a.steps):
            b.copy_(b_host, non_blocking=True)
            step()
            x_host.copy_(x, non_blocking=True)
        f1.record(stream)
        f1.synchronize()
        ms_e2e = f0.elapsed_time(f1) / a.steps
        t = torch.tensor([ms, ms_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e = (float(v) for v in t)
        # gather X to rank 0 (padded to the largest slab)
        rmax = max(bounds[q + 1] - bounds[q] for q in range(world))
        plane = int(np.prod(dims[:-1]))
        slot = torch.zeros(rmax * plane, dtype=torch.float64, device=dev)
        slot[: x.numel()].copy_(x)
        allx = torch.empty(world * rmax * plane, dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(allx, slot)
        torch.cuda.synchronize()
    res = None
    if rank == 0:
        g = allx.cpu().numpy()
        parts = []
        for q in range(world):
            rows = bounds[q + 1] - bounds[q]
            seg = g[q * rmax * plane:q * rmax * plane + rows * plane]
            parts.append(seg.reshape(tuple(dims[:-1]) + (rows,), order="F"))
        xs = np.concatenate(parts, axis=len(dims) - 1)
        res = T.residual(p, xs)
        tr_f, solve_f = flops_alg(kind, dims)
        if mode == "decoupled":
            par = (f"{world} slabs along mode {len(dims) - 1} (rows {bounds}) for the transforms of "
                   f"modes 0..{len(dims) - 2}, {world} slabs along mode 0 (rows {be.b0}) for the mode-"
                   f"{len(dims) - 1} transforms and the fibre solve along mode {be.f}; two NCCL "
                   f"all-to-alls per solve, each pipelined in {len(be.cb) - 1} chunk(s) of the slab "
                   "against the neighbouring chunks' transforms")
            # our kernels per step: phase A/C transforms (<= d-1 passes each way) + phase B
            # (state reset, mode-(d-1) transform, fibre solve, back transform)
            # + the re-sharding pack and unpack kernels (tsg_slab_pack), one each per chunk
            launches = a.steps * ((2 * (len(dims) - 1) + 2) * (len(be.cb) - 1) + 4)
        else:
            par = (f"{world} slabs along mode {len(dims) - 1} (rows {bounds}); NCCL all-gather for the "
                   "last-mode transforms, peer-mapped dataflow solve")
            launches = 7 * a.steps
        line = {
            "metric": METRIC, "value": N / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": max(a.warmup, 3), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded RandomStream, BASELINE.json distributions)",
            "config": config_of(a.config),
            "details": {"l2": "inputs larger than L2 (8N bytes per tensor > 126 MB L2)",
                        "parallelism": par, "sharded_path": mode,
                        "schur_setup": "host LAPACK dgees, outside the timed region"},
            "fp64_tflops_alg": (tr_f + solve_f) / (ms * 1e-3) / 1e12,
            "frac_fp64_peak_alg": (tr_f + solve_f) / (ms * 1e-3) / 1e12 / PEAK_FP64_TFLOPS / world,
            "residual": res,
            "roofline": {"bound": "tensor", "achieved": tr_f / (ms * 1e-3) / 1e12 / world,
                         "peak": PEAK_FP64_TFLOPS, "unit": "TFLOP/s",
                         "frac": tr_f / (ms * 1e-3) / 1e12 / world / PEAK_FP64_TFLOPS,
                         "traffic": None,
                         "kernel": "mode transforms (K1) per GPU, whole step incl. all-to-alls",
                         "peak_source": "measured FP64 DMMA peak, profiles/r01_fp64_peak_probe.log"},
            "e2e": {"value": N / (ms_e2e * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N, "ms_per_step": ms_e2e},
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    torch.cuda.synchronize()
    # orderly teardown: the library's stream (used by NCCL through torch's
    # ExternalStream) outlives every tensor and collective that touched it
    del slot, allx, b, x, b_host, x_host  # pinned buffers free through events on that stream
    if mode == "decoupled":
        be.close()
    del sl, be
    dist.destroy_process_group()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-all-configs", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="sharded path even at N=1")
    ap.add_argument("--chunks", type=int, default=0,
                    help="sharded path: pipeline chunks per slab (0 = 4 when N > 1, else 1)")
    ap.add_argument("--sharded-ipc", action="store_true",
                    help="multi-GPU: the tile-DAG path over peer-mapped slabs instead of the decoupled one")
    a = ap.parse_args()
    rank, world, local = dist_env()
    if a.impl == "reference":
        run_reference(a, rank)
    elif (world > 1 or a.sharded) and CONFIGS[a.config][0] != 5 and (len(CONFIGS[a.config][1]) == 3
                                                                       or not a.sharded_ipc):
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        run_sharded(a, rank, world, local)
    else:
        run_ours(a, rank, world, local)


if __name__ == "__main__":
    main()
