#!/bin/bash
# Round-2 configuration sweep: one bench.py JSON line per config into gpurun_out/configs_r02.jsonl
out=gpurun_out/configs_r02.jsonl
: > $out
run() { timeout 900 python bench.py "$@" 2>>gpurun_out/configs_r02.err | tail -1 >> $out; }
run --steps 10 --warmup 3
run --eps 1e-6 --steps 10 --warmup 3
run --shape papers100M --eps 1e-6 --steps 5 --warmup 3 --no-cpu-baseline
run --shape papers100M --eps 1e-7 --steps 5 --warmup 3 --no-cpu-baseline
run --method local-ch --steps 5 --warmup 3
run --method local-ch --problem katz --steps 5 --warmup 3
run --method local-hb --steps 5 --warmup 3
run --method local-hk --tau 10 --seeds 64 --steps 3 --warmup 3 --cpu-seconds 20
run --shape arxiv --method local-hk --tau 10 --steps 3 --warmup 3
run --shape arxiv --eps 1e-6 --steps 10 --warmup 3
run --shape arxiv --eps 5.905e-6 --steps 10 --warmup 3
run --shape arxiv --eps 1e-7 --steps 3 --warmup 3
run --shape arxiv --eps 1e-6 --method local-sor --omega 1 --steps 5 --warmup 3
run --shape arxiv --eps 1e-6 --method local-sor --omega 1.3930 --steps 3 --warmup 3
run --method local-sor --omega 1.3930 --steps 3 --warmup 3
run --shape cora --eps 1e-6 --seeds 50 --steps 10 --warmup 3
run --shape cora --eps 1e-6 --seeds 50 --method local-sor --omega 1 --steps 10 --warmup 3
echo done
