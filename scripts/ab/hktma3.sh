o=gpurun_out/hktma_ab3.txt; : > $o
cfg="--shape arxiv --method local-hk --tau 10 --steps 3 --warmup 3"
for i in 1 2; do
for v in AUTO 0 1; do
  if [ $v = AUTO ]; then e="X=1"; else e="GDIFF_HK_TMA=$v"; fi
  env $e timeout 1200 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|T$v [$cfg] |" >> $o
done; done
