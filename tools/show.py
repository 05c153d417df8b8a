"""Summarise bench JSON lines: python tools/show.py FILE... (one line per file)."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            k = {a: (round(b["ms_per_step"], 4), b.get("avg_launch_us"), b.get("hbm_gbs"))
                 for a, b in d.get("kernels", {}).items()}
            print(f.split("/")[-1], "ms", d["ms_per_step"], "val", d["value"], "roof",
                  d.get("roofline", {}).get("frac"), d.get("roofline", {}).get("kernel"),
                  "step", d.get("step_roofline", {}).get("frac"))
            for a, b in k.items():
                print("   ", a, b)
