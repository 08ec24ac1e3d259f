"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file X) into
per-kernel launch counts, average durations and shares: launch_summary.py X.csv OUT.json"""
import csv, json, sys
from collections import OrderedDict

src, out = sys.argv[1], sys.argv[2]
lines = open(src).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(lines[start:]))
agg = OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    us = v / 1e3 if r["Metric Unit"] == "ns" else (v * 1e3 if r["Metric Unit"] == "ms" else v)
    k = r["Kernel Name"]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
ks = sorted(agg.items(), key=lambda kv: -kv[1][1])
json.dump({"command": " ".join(sys.argv[3:]) or "ncu --metrics gpu__time_duration.sum --clock-control none",
           "launches": sum(a[0] for a in agg.values()), "total_us": round(tot, 1),
           "kernels": [{"kernel": k, "launches": a[0], "avg_us": round(a[1] / a[0], 2),
                        "share_pct": round(100 * a[1] / tot, 2)} for k, a in ks]},
          open(out, "w"), indent=1)
print(json.dumps([(k[:60], a[0], round(100 * a[1] / tot, 1)) for k, a in ks[:8]], indent=0))
