timeout 1500 python -m pytest tests/test_gpu_signed.py tests/test_gpu_xparity.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/stail_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/stail_tests.log
o=gpurun_out/stail_ab.txt; : > $o
for cfg in "--method local-ch --problem katz --steps 5 --warmup 3" "--method local-ch --steps 3 --warmup 3" "--method local-hb --steps 3 --warmup 3"; do
  GDIFF_TAIL=0 timeout 900 python bench.py $cfg --no-global-gd 2>>$o.err | tail -1 | sed "s|^|OFF [$cfg] |" >> $o
  timeout 900 python bench.py $cfg --no-global-gd 2>>$o.err | tail -1 | sed "s|^|NEW [$cfg] |" >> $o
done
