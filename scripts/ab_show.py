"""Summarise an A/B file written by scripts/ab.sh."""
import json, re, sys
for l in open(sys.argv[1]):
    m = re.match(r"(\S+) \[(.*?)\] (.*)", l)
    if not m:
        continue
    try:
        d = json.loads(m.group(3))
    except Exception:
        print(m.group(1), m.group(2), "BAD", m.group(3)[:200]); continue
    print(f"{m.group(1):5s} {m.group(2):45s} {d['value']:10.1f} {d['unit']} ms/step {d['ms_per_step']:8.3f} "
          f"kern {d['roofline'].get('kernel_ms_per_step', 0):8.3f} e2e {d['e2e']['value'] if d.get('e2e') else 0:10.1f}")
