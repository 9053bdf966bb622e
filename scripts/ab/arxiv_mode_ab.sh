o=gpurun_out/arxiv_mode_ab.txt; : > $o
for cfg in "--shape arxiv --eps 1e-6 --steps 10 --warmup 3" "--shape arxiv --eps 1e-7 --steps 3 --warmup 3" "--shape arxiv --eps 5.905e-6 --steps 10 --warmup 3"; do
  timeout 900 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|CTA [$cfg] |" >> $o
  GDIFF_BATCH_MODE=rounds timeout 900 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|ROUNDS [$cfg] |" >> $o
done
