o=gpurun_out/katz_slots2.txt; : > $o
cfg="--method local-ch --problem katz --steps 5 --warmup 3 --no-cpu-baseline --no-global-gd"
for sl in 256 512 1024; do
  GDIFF_TAIL_MEM_GB=64 timeout 900 python bench.py $cfg --slots $sl 2>>$o.err | tail -1 | sed "s|^|T_S$sl [katz] |" >> $o
  GDIFF_TAIL=0 timeout 900 python bench.py $cfg --slots $sl 2>>$o.err | tail -1 | sed "s|^|N_S$sl [katz] |" >> $o
done
