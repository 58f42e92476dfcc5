"""Summarise an ncu source-page CSV (SASS view) by instruction region:
stall-reason samples per region and the hottest instructions.
usage: python tools/sass_regions.py <sass.csv> [region_size]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
B = int(sys.argv[2]) if len(sys.argv) > 2 else 200
hdr, data = rows[1], rows[2:]
isrc = hdr.index("Source")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {r: hdr.index(r) for r in reasons}
tot = sum(float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0) for r in data)
print(f"instructions {len(data)}  samples {tot:.0f}")
for s in range(0, len(data), B):
    agg = {r: sum(float(d[idx[r]] or 0) for d in data[s:s + B]) for r in reasons}
    t = sum(agg.values())
    if t / tot < 0.01:
        continue
    top = sorted(agg.items(), key=lambda kv: -kv[1])[:4]
    print(f"{s:6d} {100 * t / tot:5.1f}%  " + "  ".join(f"{k[6:]}={100 * v / tot:.1f}" for k, v in top),
          "|", data[s][isrc][:40])
