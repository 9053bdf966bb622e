timeout 1800 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/init_tests.log 2>&1; tail -3 gpurun_out/init_tests.log
bash scripts/ab.sh ab_init.txt "--steps 20 --warmup 3" "--eps 1e-6 --steps 20 --warmup 3" "--shape papers100M --eps 1e-6 --steps 5 --warmup 3"
