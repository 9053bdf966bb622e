o=gpurun_out/hkvar_ab.txt; : > $o
for v in 1_14 1_20 1_28; do
for cfg in "--method local-hk --tau 10 --seeds 64 --steps 3 --warmup 3" "--shape arxiv --method local-hk --tau 10 --steps 3 --warmup 3"; do
  GDIFF_LIB=$PWD/exp/libgdiff_hk_$v.so timeout 1200 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|V$v [$cfg] |" >> $o
done; done
