"""Per-launch DRAM traffic of the GEMM engine from an `ncu --set full` capture
(the roofline `traffic` figure in bench.py):
    python tools/ncu_gemm_traffic.py capture.ncu-rep out.json
Writes every captured launch (duration, grid, DRAM bytes read + written, DMMA
pipe utilisation) and the launch-time-weighted mean traffic per launch of the
captured GEMM launches, plus the single longest launch."""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader([ln for ln in txt.splitlines() if ln.startswith('"')]))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}


def val(r, name):
    i = col.get(name)
    if i is None or i >= len(r) or r[i] in ("", "n/a"):
        return None
    v = float(r[i].replace(",", ""))
    u = units[i]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
             "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
    return v * scale


launches = []
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    if "gemm_dmma" not in name:
        continue
    rd = val(r, "dram__bytes_read.sum") or 0.0
    wr = val(r, "dram__bytes_write.sum") or 0.0
    launches.append({
        "kernel": name.split("(")[0].replace("(anonymous namespace)::", ""),
        "grid": r[col["Grid Size"]] if "Grid Size" in col else None,
        "duration_us": val(r, "gpu__time_duration.sum"),
        "dram_bytes": rd + wr,
        "dmma_pipe_pct": val(r, "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
    })
tot_t = sum(x["duration_us"] or 0.0 for x in launches)
summary = {
    "source": rep,
    "launches": len(launches),
    "traffic_bytes_per_launch_mean": sum(x["dram_bytes"] for x in launches) / max(1, len(launches)),
    "traffic_bytes_per_launch_time_weighted": sum(x["dram_bytes"] * (x["duration_us"] or 0) for x in launches)
    / max(tot_t, 1e-30),
    "longest": max(launches, key=lambda x: x["duration_us"] or 0) if launches else None,
    "all": launches,
}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in summary.items() if k != "all"}, indent=1))
