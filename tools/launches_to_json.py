"""ncu launch-list CSV (tools/profile_bench.sh) -> profiles/.../bench_launches.json
and profiles/traffic.json (DRAM bytes of one bench step: the last prep + grouped pair)."""
import csv
import json
import sys
from collections import OrderedDict

src, dst = sys.argv[1], sys.argv[2]
rows = [r for r in csv.DictReader(l for l in open(src) if l.startswith('"'))]
per = OrderedDict()
for r in rows:
    key = r["ID"]
    e = per.setdefault(key, {"kernel": r["Kernel Name"].split("(")[0].split("::")[-1]})
    v = float(r["Metric Value"].replace(",", ""))
    name = r["Metric Name"]
    unit = r.get("Metric Unit", "")
    if name == "gpu__time_duration.sum":
        e["duration_ns"] = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
    elif name.startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
        e["dram_bytes"] = e.get("dram_bytes", 0.0) + v * scale
    elif name == "launch__grid_size":
        e["grid"] = int(v)
launches = list(per.values())
json.dump({"note": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                   "--clock-control none, kernels of bench.py steps (group_prep_kernel + gemv_group_kernel), "
                   "serialised by ncu: compare shares, not absolutes",
           "command": "tools/profile_bench.sh", "launches": launches}, open(dst, "w"), indent=1)
step = launches[-2:]
print(json.dumps(step))
tot = sum(l["duration_ns"] for l in step)
print("grouped share of step:", step[-1]["duration_ns"] / tot, "dram bytes/step:", sum(l.get("dram_bytes", 0) for l in step))
