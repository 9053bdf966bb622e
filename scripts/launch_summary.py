"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {'nsecond': 1e-6, 'usecond': 1e-3, 'msecond': 1, 'ns': 1e-6, 'us': 1e-3, 'ms': 1}
for r in rows[1:]:
    if r[ki] == 'Kernel Name':
        continue
    agg[r[ki][:100]][0] += 1
    agg[r[ki][:100]][1] += float(r[vi].replace(',', '')) * scale[r[ui]]
tot = sum(v[1] for v in agg.values())
print(f"# {sys.argv[2] if len(sys.argv) > 2 else ''}")
print(f"# total {tot:.2f} ms over {sum(v[0] for v in agg.values())} launches")
for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{ms:10.3f} ms {100 * ms / tot:6.2f}% {c:7d} launches  {k}")
