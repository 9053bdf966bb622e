timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py -x -q -m gpu -k "products or rmat or waves" > gpurun_out/hg_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/hg_tests.log
bash scripts/ab.sh ab_hubgrp.txt "--steps 20 --warmup 3" "--eps 1e-6 --steps 20 --warmup 3" "--shape papers100M --eps 1e-7 --steps 5 --warmup 3"
