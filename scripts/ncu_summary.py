"""Summarise an ncu report: SOL / memory / occupancy numbers + top stall lines."""
import csv
import subprocess
import sys

rep = sys.argv[1]
KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Achieved Occupancy", "Registers Per Thread", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Grid Size",
        "Block Size", "Compute (SM) Throughput")
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
idx = {h: i for i, h in enumerate(r[0])}
seen = set()
for row in r[1:]:
    name = row[idx["Metric Name"]]
    if name in KEEP and name not in seen:
        seen.add(name)
        print(f"{name:40s} {row[idx['Metric Value']]:>14s} {row[idx['Metric Unit']]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
if len(rr) > 2:
    h = rr[0]
    for want in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                 "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum", "lts__t_requests_srcunit_tex_op_atom.sum"):
        if want in h:
            j = h.index(want)
            print(f"{want:40s} {rr[2][j]:>14s} {rr[1][j]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
col = "Warp Stall Sampling (All Samples)"
tot = sum(float(x[ix[col]] or 0) for x in data) or 1.0
print("top stall sites (% of samples):")
for x in sorted(data, key=lambda x: -float(x[ix[col]] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
    print(f"  {100 * float(x[ix[col]] or 0) / tot:5.1f}%  {x[ix['Source']][:100]}")
