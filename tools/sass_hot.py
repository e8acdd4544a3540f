"""Hot SASS of one kernel in an ncu report: instruction-count groups and the
top stall-sampled instructions (ncu --page source --csv)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
iSrc, iA = h.index("Source"), h.index("Address")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[iS] or 0), int(r[iE] or 0), r[iA], r[iSrc]))
    except (ValueError, IndexError):
        pass
ts, te = sum(d[0] for d in data), sum(d[1] for d in data)
print(f"samples {ts}  instructions {te / 1e6:.1f}M")
g = collections.defaultdict(lambda: [0, 0, 0])
for s, e, _, _ in data:
    g[e][0] += 1
    g[e][1] += e
    g[e][2] += s
for e, v in sorted(g.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  exec/instr {e:10d}  #instr {v[0]:5d}  {v[1] / 1e6:8.1f}M ({100 * v[1] / te:4.1f}%)  samples {100 * v[2] / max(ts, 1):4.1f}%")
for d in sorted(data, key=lambda x: -x[0])[:top]:
    print(f"{d[0]:7d} {100 * d[0] / max(ts, 1):5.1f}% {d[1]:10d} {d[3][:90]}")
