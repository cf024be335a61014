"""profiles/traffic.json from an ncu launch list of the bench step (group_prep_kernel
+ gemv_group_kernel DRAM read+write bytes per step), stamped with the hash of the
kernel sources it was captured on (bench.py reports it only while that matches).
  python tools/traffic_json.py gpurun_out/launches.csv"""
import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.DictReader(lines))
k = defaultdict(dict)
for r in rows:
    k[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    k[r["ID"]]["name"] = r["Kernel Name"]
ids = sorted(k, key=int)
# the last complete (prep, group) pair of the capture = one bench step
steps = [(a, b) for a, b in zip(ids, ids[1:])
         if k[a]["name"].startswith("group_prep") and k[b]["name"].startswith("qigen::gemv_group")
         or (k[a]["name"].startswith("group_prep") and "gemv_group_kernel" in k[b]["name"])]
a, b = steps[-1]
dram = sum(k[i]["dram__bytes_read.sum"] + k[i]["dram__bytes_write.sum"] for i in (a, b))
out = {"dram_bytes_per_step": dram, "algorithmic_bytes_per_step": bench.STEP_BYTES,
       "gemv_group_kernel_dram_bytes": k[b]["dram__bytes_read.sum"] + k[b]["dram__bytes_write.sum"],
       "gemv_group_kernel_us": k[b]["gpu__time_duration.sum"] / 1e3 if k[b]["gpu__time_duration.sum"] > 1e4 else k[b]["gpu__time_duration.sum"],
       "kernel_sources_sha16": bench._kernel_sources_sha16(),
       "source": sys.argv[1]}
(ROOT / "profiles" / "traffic.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
