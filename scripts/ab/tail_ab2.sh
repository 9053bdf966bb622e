timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/tail_tests2.log 2>&1; tail -3 gpurun_out/tail_tests2.log
o=gpurun_out/tail_ab2.txt; : > $o
for cfg in "--shape papers100M --eps 1e-6 --steps 5 --warmup 3" "--shape papers100M --eps 1e-7 --steps 5 --warmup 3" "--steps 20 --warmup 3"; do
for i in 1 2; do
  GDIFF_TAIL=0 timeout 900 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|OFF [$cfg] |" >> $o
  timeout 900 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|NEW [$cfg] |" >> $o
done; done
