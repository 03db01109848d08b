"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(d["Metric Unit"], 1.0)
        k = d["Kernel Name"].split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale
tot = sum(v[1] for v in agg.values())
steps = int(sys.argv[2]) if len(sys.argv) > 2 else max(1, agg.get("k_combine", [1])[0])
print(f"total {tot:.3f} ms over {steps} step(s)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{v[1] / steps:9.3f} ms/step {v[0]:5d} launches {100 * v[1] / tot:5.1f}%  {k}")
