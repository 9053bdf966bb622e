#!/bin/bash
# slot-count / relabel sweep of the batched kernel (products shape, eps 1e-7)
cd "$(dirname "$0")/.."
for rl in ${RL:-""}; do
for s in ${SLOTLIST:-8 16 32 64 128 256}; do
  python bench.py --steps 2 --warmup 1 --seeds 256 --slots $s --no-cpu-baseline --no-e2e $rl "$@" 2>&1 | tail -1 | \
   python -c "import json,sys; d=json.loads(sys.stdin.read()); print('slots',$s,'relabel','$rl', 'solves/s %.0f'%d['value'], 'gteps %.2f'%d['gteps'], 'kern_ms/step %.2f'%d['roofline']['kernel_ms_per_step'], 'ms/step %.2f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'])" || echo "slots $s failed"
done; done
