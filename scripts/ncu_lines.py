"""Stall samples aggregated by CUDA source line (ncu --print-source cuda,sass)."""
import csv, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = defaultdict(float); text = {}
cur = None; fname = ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 5 or r[0] == "Line No":
        continue
    if r[0]:
        cur = (fname, r[0]); text[cur] = r[1]
    try:
        v = float(r[4] or 0)
    except ValueError:
        continue
    if cur:
        agg[cur] += v
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100*v/tot:5.1f}%  {k[0]}:{k[1]:>4}  {text[k].strip()[:100]}")
