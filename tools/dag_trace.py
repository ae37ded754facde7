"""Summarise a QDWHG_DAG_TRACE file (last launch): per-task-type durations,
dependency waits, and the leaf chain.  python tools/dag_trace.py trace.txt"""
import sys
from collections import defaultdict

rows, lrows, cur, lcur = [], [], None, None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur, lcur = [], []
        rows.append(cur)
        lrows.append(lcur)
        continue
    if line.startswith("L "):
        lcur.append([int(x) for x in line.split()[1:]])
        continue
    cur.append([int(x) for x in line.split()])
last = rows[-1]
t0 = min(r[6] for r in last)
t1 = max(r[8] for r in last)
print(f"tasks {len(last)}  span {(t1 - t0) / 1e3:.1f} us")
names = {0: "leaf", 1: "panel", 2: "update", 3: "acc", 4: "fin"}
agg = defaultdict(lambda: [0, 0.0, 0.0])
for r in last:
    key = (names[r[0]], r[5])
    a = agg[key]
    a[0] += 1
    a[1] += (r[8] - r[7]) / 1e3
    a[2] += (r[7] - r[6]) / 1e3
mhz = [r[10] / max(1, r[8] - r[7]) * 1e3 for r in last if len(r) > 10 and r[8] > r[7]]
if mhz:
    mhz.sort()
    print(f"effective SM clock over tasks: median {mhz[len(mhz) // 2]:.0f} MHz (p10 {mhz[len(mhz) // 10]:.0f}, p90 {mhz[9 * len(mhz) // 10]:.0f})")
for k, (n, run, wait) in sorted(agg.items()):
    print(f"{k[0]:7s} nr={k[1]:3d} n={n:6d} run avg {run / n:7.2f} us  wait avg {wait / n:7.2f} us  run total {run:9.1f}")
busy = sum((r[8] - r[7]) for r in last) / 1e3
sms = len(set(r[9] for r in last))
print(f"busy {busy:.1f} us over {sms} SMs -> utilisation {busy / sms / ((t1 - t0) / 1e3):.2f}")
leaves = sorted([r for r in last if r[0] == 0], key=lambda r: r[3])
prev_end = None
for r in leaves[: 6] + leaves[-3:]:
    gap = (r[7] - prev_end) / 1e3 if prev_end else 0.0
    print(f"leaf k={r[3]:3d} grab {(r[6] - t0) / 1e3:8.1f} ready {(r[7] - t0) / 1e3:8.1f} "
          f"end {(r[8] - t0) / 1e3:8.1f} run {(r[8] - r[7]) / 1e3:6.1f}")
    prev_end = r[8]
# gaps between consecutive leaves: leaf(k) end -> leaf(k+1) ready
g = [(leaves[i + 1][7] - leaves[i][8]) / 1e3 for i in range(len(leaves) - 1)]
lr = [(l[8] - l[7]) / 1e3 for l in leaves]
print(f"leaf run total {sum(lr):.1f} us, inter-leaf gaps total {sum(g):.1f} us "
      f"(mean {sum(g) / max(1, len(g)):.1f}, max {max(g) if g else 0:.1f})")
late = [(leaves[i + 1][7] - leaves[i + 1][6]) / 1e3 for i in range(len(leaves) - 1)]
print("leaf grab->ready waits (first 10):", " ".join(f"{x:.0f}" for x in late[:10]))
grab_late = [(leaves[i + 1][6] - leaves[i][8]) / 1e3 for i in range(len(leaves) - 1)]
print("leaf(k+1) grab - leaf(k) end (first 16):", " ".join(f"{x:.0f}" for x in grab_late[:16]))

lt = lrows[-1]
if lt:
    ready = {r[3]: r[7] for r in last if r[0] == 0}
    ph = [[(l[1] - ready[l[0]]) / 1e3, (l[2] - l[1]) / 1e3, (l[3] - l[2]) / 1e3, (l[4] - l[3]) / 1e3] for l in lt]
    n = len(ph)
    print("leaf phases avg (load, factor, invert, write): " +
          " ".join(f"{sum(p[i] for p in ph) / n:.1f}" for i in range(4)) + " us")
