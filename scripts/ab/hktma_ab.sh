o=gpurun_out/hktma_ab.txt; : > $o
for cfg in "--method local-hk --tau 10 --seeds 64 --steps 3 --warmup 3" "--shape arxiv --method local-hk --tau 10 --steps 3 --warmup 3"; do
for i in 1 2; do
  GDIFF_HK_TMA=0 timeout 1200 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|LDG [$cfg] |" >> $o
  timeout 1200 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|TMA [$cfg] |" >> $o
done; done
