o=gpurun_out/stagecap_ab.txt; : > $o
for cfg in "--steps 20 --warmup 3" "--eps 1e-6 --steps 20 --warmup 3" "--shape papers100M --eps 1e-7 --steps 5 --warmup 3"; do
for i in 1 2; do
  GDIFF_LIB=$PWD/exp/libgdiff_head.so timeout 900 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|S3072 [$cfg] |" >> $o
  GDIFF_LIB=$PWD/exp/libgdiff_sc6144.so timeout 900 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|S6144 [$cfg] |" >> $o
done; done
