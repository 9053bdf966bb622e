set -x
o=gpurun_out/ab_overlap.jsonl; : > $o
for i in 1 2; do
 GDIFF_LIB=$PWD/exp/libgdiff_head.so timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>>gpurun_out/ab.err | tail -1 | sed 's/^/HEAD /' >> $o
 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>>gpurun_out/ab.err | tail -1 | sed 's/^/NEW /' >> $o
done
timeout 900 python bench.py --shape papers100M --eps 1e-6 --steps 5 --warmup 3 --no-cpu-baseline 2>>gpurun_out/ab.err | tail -1 | sed 's/^/PAPERS6 /' >> $o
timeout 900 python bench.py --shape papers100M --eps 1e-7 --steps 5 --warmup 3 --no-cpu-baseline 2>>gpurun_out/ab.err | tail -1 | sed 's/^/PAPERS7 /' >> $o
