"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total and mean duration, share of all kernel time.
python tools/launch_summary.py launches.csv [top]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = [ln for ln in open(path) if ln.startswith('"')]
rd = csv.DictReader(rows)
agg = defaultdict(lambda: [0, 0.0])
for r in rd:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("qdwhg::", "").replace("<unnamed>::", "")
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
    a = agg[name]
    a[0] += 1
    a[1] += v * scale
tot = sum(v[1] for v in agg.values())
n = sum(v[0] for v in agg.values())
print(f"{n} launches, {tot / 1e3:.2f} ms total kernel time (serialised, cold-cache ncu replay)")
print(f"{'share':>6} {'total ms':>9} {'count':>6} {'mean us':>9}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{100 * v[1] / tot:5.1f}% {v[1] / 1e3:9.3f} {v[0]:6d} {v[1] / v[0]:9.1f}  {k[:90]}")
