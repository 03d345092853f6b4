#!/usr/bin/env python
"""Summarise an ncu --set full report of the daemon kernel + the launch list into
profiles/ (key SOL metrics, DRAM/L2 traffic, stall mix) -- run here, no GPU."""
import csv
import io
import json
import subprocess
import sys

rep, launches, out = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum"]
res = {}
for i, h in enumerate(hdr):
    if h in want:
        res[h] = (vals[i], units[i])
lines = ["# ncu --set full summary of occl_daemon_kernel (1 launch, bench config, 2 steps)", ""]
for k in want:
    if k in res:
        lines.append(f"{k:60s} {res[k][0]} {res[k][1]}")
# launch list
lcsv = open(launches).read().splitlines()
start = next(i for i, l in enumerate(lcsv) if l.startswith('"ID"'))
lr = list(csv.DictReader(io.StringIO("\n".join(lcsv[start:]))))
tot = {}
for r in lr:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ns = v * (1e6 if unit == "ms" else 1e3 if unit in ("us", "usecond") else 1.0)
        k = r["Kernel Name"].split("(")[0][:60]
        tot[k] = tot.get(k, 0.0) + ns
lines += ["", "# launch list (ncu gpu__time_duration, cold + serialised: compare shares)", ""]
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    lines.append(f"{k:60s} {v/1e6:10.3f} ms  {100*v/T:5.1f}%")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
d = float(res["dram__bytes_read.sum"][0]) + float(res["dram__bytes_write.sum"][0])
mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[res["dram__bytes_read.sum"][1]]
print(json.dumps({"dram_bytes_per_launch": d * mult}))
