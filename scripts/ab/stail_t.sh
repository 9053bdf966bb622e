o=gpurun_out/stail_t.txt; : > $o
cfg="--method local-ch --problem katz --steps 5 --warmup 3 --no-cpu-baseline --no-global-gd"
for tt in 16 8 4 2 1; do
  GDIFF_TAIL_T=$tt timeout 900 python bench.py $cfg 2>>$o.err | tail -1 | sed "s|^|T$tt [katz] |" >> $o
done
GDIFF_TAIL_T=4 GDIFF_TAIL_F=65536 timeout 900 python bench.py $cfg 2>>$o.err | tail -1 | sed "s|^|T4F64K [katz] |" >> $o
