python scripts/hk_rounds_probe.py arxiv > gpurun_out/hk_rounds_arxiv2.txt 2>&1
python scripts/hk_rounds_probe.py products > gpurun_out/hk_rounds_products2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q -m gpu -k hk > gpurun_out/hk_t2.log 2>&1; tail -1 gpurun_out/hk_t2.log
