o=gpurun_out/gm_ab.txt; : > $o
for i in 1 2; do
for gm in 4194304 2000000 1000000 500000; do
  GDIFF_GROUP_MIN=$gm timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|GM$gm [products 1e-7] |" >> $o
done; done
for gm in 4194304 1000000; do
  GDIFF_GROUP_MIN=$gm timeout 600 python bench.py --eps 1e-6 --steps 20 --warmup 3 --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|GM$gm [products 1e-6] |" >> $o
  GDIFF_GROUP_MIN=$gm timeout 900 python bench.py --shape papers100M --eps 1e-6 --steps 5 --warmup 3 --no-cpu-baseline --no-global-gd 2>>$o.err | tail -1 | sed "s|^|GM$gm [papers 1e-6] |" >> $o
done
