#!/bin/bash
# round-2 final evidence: tests, smoke, bench (both arms), launch list, ncu captures
cd "$(dirname "$0")/.."
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/final_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-global-gd > gpurun_out/ncu_launch_final.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^k_rounds$|k_rounds<|k_tail" -s 40 -c 2 \
  -o gpurun_out/prof_final python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-global-gd > gpurun_out/ncu_full_final.log 2>&1; echo "ncu full rc=$?"
