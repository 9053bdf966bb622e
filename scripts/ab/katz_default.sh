timeout 1500 python -m pytest tests/test_gpu_signed.py tests/test_gpu_xparity.py -x -q -m gpu -k "ch or katz or hb or signed" > gpurun_out/kd_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/kd_tests.log
o=gpurun_out/katz_default.txt; : > $o
for cfg in "--method local-ch --problem katz --steps 5 --warmup 3" "--method local-ch --steps 3 --warmup 3" "--method local-hb --steps 3 --warmup 3"; do
  timeout 900 python bench.py $cfg --no-global-gd 2>>$o.err | tail -1 | sed "s|^|NEW [$cfg] |" >> $o
done
