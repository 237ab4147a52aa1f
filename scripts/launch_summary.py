"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into per-kernel counts, time and share."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0]
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"]) * (1e-3 if d.get("Metric Unit") == "ns" else 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>6s}  kernel")
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:8d} {us:12.1f} {us / n:10.1f} {100 * us / tot:5.1f}%  {k}")
