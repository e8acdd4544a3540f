"""Summarise ncu reports into profiles/ (text) and the dominant kernel's DRAM
traffic per launch into profiles/ncu_traffic.json (read by bench.py)."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        # the tensor-pipe counters that see mma.sync.f64 (DMMA); the fp64 pipe ones do not
        "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:80]}
        for k in KEYS:
            if k in h:
                d[k] = f"{r[h.index(k)]} {units[h.index(k)]}".strip()
        res.append(d)
    return res


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def to_bytes(s):
    v, _, u = s.partition(" ")
    return float(v.replace(",", "")) * SCALE.get(u.strip(), 1)


def main():
    out_txt, config = sys.argv[1], sys.argv[2]
    reps = sys.argv[3:]
    lines, traffic = [], None
    for rep in reps:
        for d in raw(rep):
            lines.append(f"== {rep}: {d['kernel']}")
            for k in KEYS:
                if k in d:
                    lines.append(f"   {k:70s} {d[k]}")
            try:
                t = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
                kind = "solve" if "solve" in d["kernel"] else ("dgemm" if "dgemm" in d["kernel"] else None)
                if kind:
                    traffic = traffic or {}
                    traffic.setdefault(kind, t)
            except (KeyError, ValueError):
                pass
    open(out_txt, "w").write("\n".join(lines) + "\n")
    if traffic is not None:
        path = "profiles/ncu_traffic.json"
        try:
            js = json.load(open(path))
        except (OSError, ValueError):
            js = {}
        js.setdefault(config, {}).update(traffic)
        json.dump(js, open(path, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
