"""Aggregate ncu warp-stall samples per CUDA source line from an .ncu-rep
(`ncu -i X --page source --csv --print-source cuda,sass`)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
agg = defaultdict(float)
srcline = {}
cur = None
hdr = None
for r in rows:
    if not r:
        continue
    if "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        i_s = r.index("Warp Stall Sampling (All Samples)")
        i_src = r.index("Source")
        continue
    if hdr is None or len(r) <= i_s:
        continue
    # cuda,sass view: CUDA source lines have a line number in column 0 (no 0x address)
    if r[0] and r[0] not in ("File Path", "Function Name"):
        cur = (r[0], r[1].strip()[:100])
        v = r[i_s]
        try:
            agg[cur] += float(v)
        except ValueError:  # "-" or a source line whose quotes broke the CSV
            pass
tot = sum(agg.values()) or 1.0
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}%  L{k[0]:>5}  {k[1]}")
