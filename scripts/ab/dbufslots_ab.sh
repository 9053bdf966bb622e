o=gpurun_out/dbufslots_ab.txt; : > $o
for cfg in "--shape papers100M --eps 1e-7 --steps 5 --warmup 3" "--shape papers100M --eps 1e-6 --steps 5 --warmup 3"; do
for i in 1 2; do
  timeout 900 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|DEF [$cfg] |" >> $o
  GDIFF_DBUF_SLOTS=1 timeout 900 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|DBS [$cfg] |" >> $o
done; done
