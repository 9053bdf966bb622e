#!/bin/bash
# BASELINE.json configs 1-2 as bench lines (run under gpurun)
cd "$(dirname "$0")/.."
run() { python bench.py "$@" --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; cb=d['cpu_baseline'] or {}
print(f\"{c['workload'][:90]:90s} | {d['value']:10.0f} solves/s | {d['gteps']:6.2f} GTEPS | frac {d['roofline']['frac']:.3f} | cpu {cb.get('value',0):8.1f}/s x{d['value']/max(cb.get('value',1e-9),1e-9):7.1f} parity={cb.get('parity_sweeps_ops_identical')}\")"; }
run --shape cora --eps 1e-6 --seeds 50 --steps 5 --warmup 3 --cpu-seconds 5
run --shape arxiv --eps 1e-6 --seeds 1024 --steps 5 --warmup 3 --cpu-seconds 10
run --shape arxiv --eps 1e-6 --seeds 1024 --steps 5 --warmup 3 --cpu-seconds 10 --method local-sor --omega 1.0
run --shape arxiv --eps 1e-6 --seeds 1024 --steps 5 --warmup 3 --cpu-seconds 10 --method local-sor --omega 1.3930115503199288
run --shape arxiv --eps 5.905e-6 --seeds 1024 --steps 5 --warmup 3 --cpu-seconds 10
run --shape products --eps 1e-6 --seeds 1024 --steps 5 --warmup 3 --cpu-seconds 10
run --shape products --eps 1e-7 --seeds 1024 --steps 5 --warmup 3 --cpu-seconds 10 --method local-sor --omega 1.3930115503199288
