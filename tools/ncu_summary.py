"""Summaries of a profile_round.sh capture for profiles/:
  python tools/ncu_summary.py gpurun_out/<tag> profiles/<name>.json [report.ncu-rep]
writes the json (per captured kernel: duration, DRAM bytes and
%, L2 %, active vs elapsed cycles, instructions, issue %, warps active,
registers, grid, top stalls) and prints the launch-list share table of
<tag>/launches.csv (gpu__time_duration / dram bytes per kernel)."""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

tag, prefix = sys.argv[1], sys.argv[2]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size"]
import os

rep = sys.argv[3] if len(sys.argv) > 3 else f"{tag}/prof.ncu-rep"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
out = []
for row in rows[2:]:
    e = {"kernel": row[h.index("Kernel Name")].split("(")[0]}
    for k in KEYS:
        if k in h:
            e[k] = row[h.index(k)]
    stalls = []
    for i, k in enumerate(h):
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", k)
        if m:
            try:
                stalls.append((m.group(1), round(float(row[i]), 2)))
            except ValueError:
                pass
    e["top_stalls"] = sorted(stalls, key=lambda x: -x[1])[:4]
    out.append(e)
json.dump(out, open(prefix, "w"), indent=1)
print(f"wrote {prefix} ({len(out)} kernels)")

# launch-list shares
if not os.path.exists(f"{tag}/launches.csv"):
    sys.exit(0)
tot = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
with open(f"{tag}/launches.csv") as fh:
    lines = [l for l in fh if l.startswith('"')]
r = list(csv.reader(lines))
hh = r[0]
ki, mi, vi = hh.index("Kernel Name"), hh.index("Metric Name"), hh.index("Metric Value")
idi = hh.index("ID")
per = defaultdict(dict)
for row in r[1:]:
    per[(row[idi], row[ki].split("(")[0])][row[mi]] = float(row[vi].replace(",", ""))
for (_i, k), mets in per.items():
    t = tot[k]
    t[0] += 1
    t[1] += mets.get("gpu__time_duration.sum", 0.0)
    t[2] += mets.get("dram__bytes_read.sum", 0.0)
    t[3] += mets.get("dram__bytes_write.sum", 0.0)
allt = sum(v[1] for v in tot.values())
print("| kernel | launches | share | avg us | avg DRAM read MB | avg DRAM write MB |")
print("|---|---|---|---|---|---|")
for k, (n, t, rd, wr) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {n} | {t / allt:.3f} | {t / n / 1e3:.1f} | {rd / n / 1e6:.1f} | {wr / n / 1e6:.1f} |")
