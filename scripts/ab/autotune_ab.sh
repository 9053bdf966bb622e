timeout 1800 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py tests/test_bench_contract.py -x -q -m gpu > gpurun_out/at_tests.log 2>&1; tail -2 gpurun_out/at_tests.log
o=gpurun_out/autotune.txt; : > $o
for cfg in "--shape arxiv --eps 1e-6 --steps 10 --warmup 3" "--shape arxiv --eps 1e-7 --steps 3 --warmup 3" "--shape arxiv --eps 5.905e-6 --steps 10 --warmup 3" "--shape cora --eps 1e-6 --seeds 50 --steps 10 --warmup 3"; do
  timeout 900 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|AUTO [$cfg] |" >> $o
done
