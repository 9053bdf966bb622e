"""Markdown table of a configs JSONL (one bench.py line per config) for DESIGN.md §6."""
import json
import sys

print("| config | GPU (device-timed) | e2e (host API) | roofline frac | CPU port (16 thr) | GPU / CPU | x parity (max rel l1, top-100 identical) |")
print("|---|---|---|---|---|---|---|")
for l in open(sys.argv[1]):
    d = json.loads(l)
    c = d["config"]["workload"].replace("batched ", "").split(", R-MAT ")
    shape = c[1].split(" (")[0] if len(c) > 1 else ""
    seeds = d["config"].get("seeds_per_gpu_per_step")
    cb = d.get("cpu_baseline") or {}
    cpu = cb.get("value")
    par = (f"{cb['x_l1_rel_max']:.1e}, {cb['topk_identical_up_to_ties']}/{cb['sample'].split()[0]}"
           if cb else "—")
    print(f"| {c[0]} {shape}, {seeds} seeds | {d['value']:,.1f} /s | {d['e2e']['value']:,.1f} /s | "
          f"{d['roofline']['frac']:.3f} | {cpu:,.1f} /s | {d['value'] / cpu:,.1f} | {par} |"
          if cpu else
          f"| {c[0]} {shape}, {seeds} seeds | {d['value']:,.1f} /s | {d['e2e']['value']:,.1f} /s | "
          f"{d['roofline']['frac']:.3f} | — | — | — |")
