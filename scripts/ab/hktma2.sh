timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py -x -q -m gpu -k "hk or heat" > gpurun_out/hktma_t3.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/hktma_t3.log
o=gpurun_out/hktma_ab2.txt; : > $o
for cfg in "--method local-hk --tau 10 --seeds 64 --steps 3 --warmup 3" "--shape arxiv --method local-hk --tau 10 --steps 3 --warmup 3"; do
  timeout 1200 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|AUTO [$cfg] |" >> $o
done
