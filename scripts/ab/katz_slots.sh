o=gpurun_out/katz_slots.txt; : > $o
cfg="--method local-ch --problem katz --steps 5 --warmup 3 --no-cpu-baseline --no-global-gd"
for sl in 64 128 256 512 1024; do
  timeout 900 python bench.py $cfg --slots $sl 2>>$o.err | tail -1 | sed "s|^|S$sl [katz] |" >> $o
done
timeout 900 python bench.py --method local-ch --steps 3 --warmup 3 --no-cpu-baseline --no-global-gd --slots 128 2>>$o.err | tail -1 | sed "s|^|S128 [ch-ppr] |" >> $o
