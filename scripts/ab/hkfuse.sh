timeout 1500 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py tests/test_gpu_parity.py -x -q -m gpu -k "hk or heat" > gpurun_out/hkf_tests.log 2>&1; tail -2 gpurun_out/hkf_tests.log
python scripts/hk_rounds_probe.py arxiv > gpurun_out/hk_rounds_arxiv3.txt 2>&1
python scripts/hk_rounds_probe.py products > gpurun_out/hk_rounds_products3.txt 2>&1
