"""Extract per-launch duration and DRAM traffic of the sweep kernel from an
ncu --set full report into profiles/<name>.json (read by bench.py)."""
import csv, json, subprocess, sys
rep, out, note = sys.argv[1], sys.argv[2], (sys.argv[3] if len(sys.argv) > 3 else "")
kernel = sys.argv[4] if len(sys.argv) > 4 else "k_rounds"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
def get(name):
    i = h.index(name)
    x = float(v[i]); unit = u[i]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1, "%": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}.get(unit, 1)
    return x * scale
d = {"kernel": kernel, "report": rep.split("/")[-1], "note": note,
     "gpu_time_s": get("gpu__time_duration.sum"),
     "dram_bytes_read": get("dram__bytes_read.sum"), "dram_bytes_write": get("dram__bytes_write.sum"),
     "l2_hit_rate_pct": get("lts__t_sector_hit_rate.pct")}
d["dram_bytes_per_launch"] = d["dram_bytes_read"] + d["dram_bytes_write"]
d["dram_gbs"] = d["dram_bytes_per_launch"] / d["gpu_time_s"] / 1e9
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d))
