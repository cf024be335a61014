"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv
--print-source sass` output, with the dominant stall reasons of each."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
k = idx["Warp Stall Sampling (All Samples)"]
ex = idx["Instructions Executed"]
stall_cols = [h for h in hdr if h.startswith("stall_")]
data = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(float(r[k] or 0) for r in data)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"total samples {tot:.0f}, instructions executed {sum(float(r[ex] or 0) for r in data):.0f}")
for r in sorted(data, key=lambda r: -float(r[k] or 0))[:n]:
    st = sorted(((float(r[idx[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{float(r[k]) / tot * 100:5.1f}% {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:60]:60s} "
          + " ".join(f"{c}:{v:.0f}" for v, c in st if v))
