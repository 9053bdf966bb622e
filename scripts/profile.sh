#!/bin/bash
# launch list + one full ncu capture of the sweep kernel (run under gpurun, 1 GPU)
cd "$(dirname "$0")/.."
ARGS="--steps 1 --warmup 1 --seeds ${SEEDS:-128} --slots ${SLOTS:-128} --no-cpu-baseline --no-e2e"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_rounds -s 1 -c 1 \
    -o gpurun_out/prof_rounds python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo "profile rc=$?"
tail -3 gpurun_out/ncu_full.log
