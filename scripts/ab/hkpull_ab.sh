timeout 1800 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py -x -q -m gpu -k "hk or heat" > gpurun_out/hkpull_tests.log 2>&1; tail -3 gpurun_out/hkpull_tests.log
o=gpurun_out/hkpull_ab.txt; : > $o
for cfg in "--method local-hk --tau 10 --seeds 64 --steps 3 --warmup 3 --cpu-seconds 20" "--shape arxiv --method local-hk --tau 10 --steps 3 --warmup 3"; do
  GDIFF_HK_PULL=0 timeout 1200 python bench.py $cfg --no-global-gd 2>>$o.err | tail -1 | sed "s|^|OFF [$cfg] |" >> $o
  timeout 1200 python bench.py $cfg --no-global-gd 2>>$o.err | tail -1 | sed "s|^|NEW [$cfg] |" >> $o
done
