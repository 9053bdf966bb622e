#!/bin/bash
# round-2 profiles: papers100M eps=1e-6 launch list of the solve kernels, and a
# full ncu capture of k_signed_rounds (LocalCH-PPR products, bench default slots)
cd "$(dirname "$0")/.."
P="--shape papers100M --eps 1e-6 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 python bench.py $P > gpurun_out/papers_plain.log 2>&1; echo "papers plain rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:"k_rounds|k_wave|k_count|k_emit" --log-file gpurun_out/launches_papers6_r02.csv \
  python bench.py $P > gpurun_out/ncu_papers.log 2>&1; echo "papers ncu rc=$?"
C="--method local-ch --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 python bench.py $C > gpurun_out/ch_plain.log 2>&1; echo "ch plain rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:"k_s|k_signed|k_pair" --log-file gpurun_out/launches_ch_r02.csv \
  python bench.py $C > gpurun_out/ncu_ch_launch.log 2>&1; echo "ch launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"^k_signed_rounds" -s 20 -c 1 \
  -o gpurun_out/prof_k_signed_rounds_r02 python bench.py $C > gpurun_out/ncu_ch_full.log 2>&1; echo "ch full rc=$?"
