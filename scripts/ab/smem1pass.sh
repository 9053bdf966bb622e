timeout 900 python -m pytest tests/test_gpu_batch.py -x -q -m gpu -k "cora or reuse or rmat_batch" > gpurun_out/s1_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/s1_tests.log
bash scripts/ab.sh ab_smem1pass.txt "--shape cora --eps 1e-6 --seeds 50 --steps 20 --warmup 3"
