timeout 1800 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py -x -q -m gpu > gpurun_out/bc_tests.log 2>&1; tail -1 gpurun_out/bc_tests.log
bash scripts/ab.sh ab_bc.txt "--steps 20 --warmup 3" "--eps 1e-6 --steps 20 --warmup 3"
