"""Summarise tools/evidence.sh output into a markdown table (profiles/):
per solve variant, the CUDA-event phase times and, per kernel family, the
ncu metrics (DMMA-pipe utilisation, FP64 pipe, DRAM traffic and bandwidth)."""
import collections
import csv
import io
import re
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02ev"
out = sys.argv[2] if len(sys.argv) > 2 else f"profiles/{tag}_solve_variants.md"
variants = ["c2_decoupled", "c2_lap16", "c2_lap3", "c3_decoupled", "c3_lapd", "c4_decoupled", "c4_lap16",
            "c5_decoupled", "c5_gsyd"]
M = {"gpu__time_duration.sum": "t", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_inst%",
     "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_cyc%",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64%",
     "dram__bytes_read.sum": "rd", "dram__bytes_write.sum": "wr",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%", "sm__warps_active.avg.pct_of_peak_sustained_active": "warps%"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0, "%": 1.0}


def family(k):
    for f in ("fibre_wide", "fibre_small", "solve_lap16", "solve_lap3", "solve_lapd", "solve_gsyd", "dgemm", "pair"):
        if f in k:
            return f
    return k[:30]


lines = ["# Solve variants: time, DMMA pipe, DRAM (tools/evidence.sh, one B200)", "",
         "Per variant: the CUDA-event phase times of `tools/perf_probe.py` (no profiler), then per kernel "
         "family the ncu metrics of one solve (`--metrics`, `--clock-control none`; per-launch averages; "
         "DMMA % = `smsp__pipe_tensor_subpipe_dmma_cycles_active` pct of peak, the tensor-pipe counter that "
         "sees `mma.sync.f64`; `sm__pipe_fp64_cycles_active` does not count DMMA).", ""]
for v in variants:
    try:
        tt = open(f"gpurun_out/{tag}_{v}_time.txt").read()
    except OSError:
        continue
    m = re.search(r"solve=(\S+).*?\n\s+fwd ([\d.]+) ms.*?solve ([\d.]+) ms.*?back ([\d.]+) ms.*?total ([\d.]+) ms", tt, re.S)
    lines.append(f"## {v}")
    if m:
        lines.append(f"kernel `{m.group(1)}`: forward {m.group(2)} ms, solve **{m.group(3)} ms**, back {m.group(4)} ms, "
                     f"total {m.group(5)} ms")
    try:
        txt = open(f"gpurun_out/{tag}_{v}_ncu.csv").read().splitlines()
        i = [k for k, l in enumerate(txt) if l.startswith('"ID"')][0]
        rows = list(csv.reader(io.StringIO("\n".join(txt[i:]))))
        h = rows[0]
        ik, im, iu, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
        agg = collections.defaultdict(lambda: collections.defaultdict(list))
        for r in rows[1:]:
            name = M.get(r[im])
            if not name:
                continue
            val = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
            agg[family(r[ik])][name].append(val)
        lines.append("")
        lines.append("| kernel | launches | avg time | DMMA cycles % | DMMA inst % | FP64 pipe % | SM % | warps % | DRAM GB/launch | DRAM GB/s |")
        lines.append("|---|---|---|---|---|---|---|---|---|---|")
        for fam, d in sorted(agg.items(), key=lambda kv: -sum(kv[1].get("t", [0]))):
            n = len(d.get("t", []))
            avg = lambda k: sum(d[k]) / len(d[k]) if d.get(k) else float("nan")
            t = avg("t")
            gb = (avg("rd") + avg("wr")) / 1e9
            lines.append(f"| {fam} | {n} | {t * 1e3:.3f} ms | {avg('dmma_cyc%'):.1f} | {avg('dmma_inst%'):.1f} | "
                         f"{avg('fp64%'):.1f} | {avg('sm%'):.1f} | {avg('warps%'):.1f} | {gb:.3f} | {gb / t:.0f} |")
    except (OSError, IndexError, ValueError) as e:
        lines.append(f"(no ncu data: {e})")
    lines.append("")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
