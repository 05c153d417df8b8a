"""Summarise bench JSON lines: python tools/show.py FILE... (one line per file)."""
import json
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)  # quiet under `| head`

for f in sys.argv[1:]:
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            k = {a: (round(b["ms_per_step"], 4), b.get("avg_launch_us"), b.get("hbm_gbs"))
                 for a, b in d.get("kernels", {}).items()}
            print(f.split("/")[-1], "ms", d["ms_per_step"], "serial", d.get("ms_per_step_serialized"), "val",
                  d["value"], "roof", d.get("roofline", {}).get("frac"), d.get("roofline", {}).get("kernel"),
                  "step", d.get("step_roofline", {}).get("frac"), "e2e", d.get("e2e", {}).get("value"))
            for a, b in k.items():
                print("   ", a, b)
            if "headline" in d:
                print("    headline", d["headline"])
