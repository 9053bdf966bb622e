#!/bin/bash
# A/B of the in-tree build against exp/libgdiff_head.so (GDIFF_LIB), alternating,
# each config twice; one tagged bench line per run into gpurun_out/$OUT
#   usage: bash scripts/ab.sh OUT "bench args 1" "bench args 2" ...
cd "$(dirname "$0")/.."
o=gpurun_out/$1; shift; : > $o
for cfg in "$@"; do
  for i in 1 2; do
    GDIFF_LIB=$PWD/exp/libgdiff_head.so timeout 900 python bench.py $cfg --no-cpu-baseline 2>>$o.err | tail -1 | sed "s|^|HEAD [$cfg] |" >> $o
    timeout 900 python bench.py $cfg --no-cpu-baseline 2>>$o.err | tail -1 | sed "s|^|NEW [$cfg] |" >> $o
  done
done
