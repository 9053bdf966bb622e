timeout 1800 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py tests/test_gpu_fullsize.py tests/test_gpu_shard.py -x -q -m gpu > gpurun_out/dbuf_tests.log 2>&1; tail -3 gpurun_out/dbuf_tests.log
o=gpurun_out/dbuf_ab.txt; : > $o
for cfg in "--steps 20 --warmup 3" "--eps 1e-6 --steps 20 --warmup 3"; do
for i in 1 2; do
  GDIFF_DBUF=0 timeout 600 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|OFF [$cfg] |" >> $o
  timeout 600 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|NEW [$cfg] |" >> $o
done; done
GDIFF_WAVE_TRACE=1 timeout 600 python scripts/wave_trace.py products 1e-7 > gpurun_out/wt_dbuf.txt 2>&1
