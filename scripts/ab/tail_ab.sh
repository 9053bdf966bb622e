# CTA-local wave tails: parity tests, then A/B (HEAD lib / new / GDIFF_TAIL=0 / thresholds)
timeout 1500 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/tail_tests.log 2>&1; tail -3 gpurun_out/tail_tests.log
o=gpurun_out/tail_ab.txt; : > $o
for cfg in "--steps 20 --warmup 3" "--eps 1e-6 --steps 20 --warmup 3"; do
for i in 1 2; do
  GDIFF_LIB=$PWD/exp/libgdiff_head.so timeout 600 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|HEAD [$cfg] |" >> $o
  timeout 600 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|NEW [$cfg] |" >> $o
  GDIFF_TAIL=0 timeout 600 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|OFF [$cfg] |" >> $o
done
for v in 8192 65536; do
  GDIFF_TAIL_P=$v timeout 600 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|P$v [$cfg] |" >> $o
done; done
