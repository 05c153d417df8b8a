import json, sys, glob
for f in sorted(glob.glob(sys.argv[1] + "/bench*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            k = {a: round(b["ms_per_step"], 4) for a, b in d.get("kernels", {}).items()}
            print(f.split("/")[-1], "ms", d["ms_per_step"], "val", d["value"], "roof", d.get("roofline", {}).get("frac"),
                  d.get("roofline", {}).get("kernel"), "step", d.get("step_roofline", {}).get("frac"), k)
