"""gpurun_out/stage_traffic_<stage>.csv (scripts/stage_traffic.sh) -> profiles/stage_traffic.json:
per stage, the number of kernel launches, summed duration and summed DRAM bytes."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
out = {"model": sys.argv[2] if len(sys.argv) > 2 else "resnet50",
       "inv_type": sys.argv[3] if len(sys.argv) > 3 else "inverse", "stages": {}}
try:
    out["commit"] = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True,
                                   text=True).stdout.strip()
except OSError:
    pass
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3,
        "second": 1.0}
for st in ("factors", "inversion", "precondition", "comm_rs", "comm_ag"):
    p = os.path.join(src, f"stage_traffic_{st}.csv")
    if not os.path.exists(p):
        continue
    text = open(p).read()
    i = text.find('"ID"')
    if i < 0:
        continue
    rows = list(csv.DictReader(io.StringIO(text[i:])))
    per = {}
    for r in rows:
        k = (r["ID"], r["Kernel Name"])
        per.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
    dram = sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in per.values())
    dur = sum(v.get("gpu__time_duration.sum", 0) for v in per.values())
    kinds = {}
    for (_, name), v in per.items():
        kn = name.split("(")[0].split("<")[0]
        a = kinds.setdefault(kn, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += v.get("gpu__time_duration.sum", 0) * 1e6
        a[2] += (v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)) / 1e6
    out["stages"][st] = {"launches": len(per), "dram_bytes": dram, "duration_ms_serialized_cold": dur * 1e3,
                         "by_kernel": {k: {"launches": a[0], "us": round(a[1], 1), "dram_MB": round(a[2], 2)}
                                       for k, a in sorted(kinds.items(), key=lambda kv: -kv[1][1])}}
dst = os.path.join(ROOT, "profiles", "stage_traffic.json")
with open(dst, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps({k: (v["launches"], round(v["dram_bytes"] / 1e6, 1), round(v["duration_ms_serialized_cold"], 3))
                  for k, v in out["stages"].items()}))
