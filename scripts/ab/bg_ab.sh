# background-reset A/B: bench ms/step on products eps=1e-7 / 1e-6 for several knobs
o=gpurun_out/bg_ab.txt; : > $o
for cfg in "--steps 20 --warmup 3" "--eps 1e-6 --steps 20 --warmup 3"; do
for env in "GDIFF_BG_RESET=0" "X=1" "GDIFF_BG_MINP=0" "GDIFF_BG_MINP=4000000" "GDIFF_BG_MINP=1000000000000" "GDIFF_BG_Q=4" "GDIFF_BG_UPW=64" "GDIFF_BG_RESET=0"; do
  env $env timeout 600 python bench.py $cfg --no-cpu-baseline 2>>$o.err | tail -1 | sed "s|^|$env [$cfg] |" >> $o
done; done
GDIFF_WAVE_TRACE=1 timeout 600 python scripts/wave_trace.py products 1e-7 > gpurun_out/wt_bg.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py tests/test_gpu_fullsize.py -x -q -m gpu 2>&1 | tail -3 >> $o
