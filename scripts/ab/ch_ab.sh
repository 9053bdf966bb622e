timeout 1500 python -m pytest tests/test_gpu_signed.py tests/test_gpu_xparity.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/ch_tests.log 2>&1; tail -3 gpurun_out/ch_tests.log
bash scripts/ab.sh ab_ch.txt "--method local-ch --steps 3 --warmup 3" "--method local-ch --problem katz --steps 3 --warmup 3" "--method local-hb --steps 3 --warmup 3"
