"""profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum per launch of each captured
kernel (from ncu --set full reports), read by bench.py for the roofline 'traffic' field."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {}
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h, units, vals = rr[0], rr[1], rr[2]
    name = vals[h.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]

    def get(k):
        v = float(vals[h.index(k)].replace(",", ""))
        u = units[h.index(k)]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

    def col(k):
        return vals[h.index(k)] if k in h else None

    dur = get("gpu__time_duration.sum") if "gpu__time_duration.sum" in h else None
    out[name] = {"dram_bytes": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
                 "dram_read": get("dram__bytes_read.sum"), "dram_write": get("dram__bytes_write.sum"),
                 "kernel": vals[h.index("Kernel Name")].split("(")[0].replace("void ", ""),
                 "grid": col("launch__grid_size"), "block": col("launch__block_size"),
                 "duration_us": None if dur is None else dur * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                                                                 "second": 1e6}.get(units[h.index("gpu__time_duration.sum")], 1.0),
                 "source": os.path.basename(rep)}
path = os.path.join(ROOT, "profiles", "traffic.json")
old = {} if os.environ.get("TRAFFIC_FRESH") else (json.load(open(path)) if os.path.exists(path) else {})
old.update(out)
json.dump(old, open(path, "w"), indent=1)
print(json.dumps(old, indent=1))
