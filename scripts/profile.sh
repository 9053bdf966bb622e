#!/bin/bash
# launch list + one full ncu capture of a sweep kernel (run under gpurun, 1 GPU)
#   KERNEL=k_rounds|k_signed_rounds  EXTRA="--method local-ch ..."  SEEDS SLOTS
cd "$(dirname "$0")/.."
K=${KERNEL:-k_rounds}
ARGS="--steps 1 --warmup 1 --seeds ${SEEDS:-128} --slots ${SLOTS:-128} --no-cpu-baseline --no-e2e ${EXTRA:-}"
python bench.py $ARGS > gpurun_out/plain_$K.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$K.csv \
    python bench.py $ARGS > gpurun_out/ncu_launch_$K.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^$K$" -s 1 -c 1 \
    -o gpurun_out/prof_$K python bench.py $ARGS > gpurun_out/ncu_full_$K.log 2>&1
echo "profile rc=$?"
tail -3 gpurun_out/ncu_full_$K.log
