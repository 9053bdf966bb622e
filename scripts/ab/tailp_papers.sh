o=gpurun_out/tailp_papers.txt; : > $o
for cfg in "--shape papers100M --eps 1e-7 --steps 5 --warmup 3" "--shape papers100M --eps 1e-6 --steps 5 --warmup 3"; do
for tp in 16384 65536 262144; do
  GDIFF_TAIL_P=$tp timeout 900 python bench.py $cfg --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|P$tp [$cfg] |" >> $o
done; done
