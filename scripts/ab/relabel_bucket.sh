GDIFF_RELABEL_BUCKET=1 timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py -x -q -m gpu -k "rmat or cora or products" > gpurun_out/rb_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/rb_tests.log
o=gpurun_out/relabel_bucket.txt; : > $o
for cfg in "--steps 20 --warmup 3" "--eps 1e-6 --steps 20 --warmup 3" "--shape papers100M --eps 1e-7 --steps 5 --warmup 3"; do
  timeout 900 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|DEG [$cfg] |" >> $o
  GDIFF_RELABEL_BUCKET=1 timeout 900 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|BKT [$cfg] |" >> $o
done
