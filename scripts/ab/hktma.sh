timeout 300 python -m pytest tests/test_gpu_batch.py -x -q -m gpu -k "hk" > gpurun_out/hktma_t1.log 2>&1; echo "small rc=$?"; tail -1 gpurun_out/hktma_t1.log
timeout 600 python -m pytest tests/test_gpu_xparity.py -x -q -m gpu -k "heat" > gpurun_out/hktma_t2.log 2>&1; echo "xparity rc=$?"; tail -1 gpurun_out/hktma_t2.log
timeout 300 python scripts/hk_rounds_probe.py arxiv > gpurun_out/hk_rounds_arxiv4.txt 2>&1; echo "probe rc=$?"
timeout 300 python scripts/hk_rounds_probe.py products > gpurun_out/hk_rounds_products4.txt 2>&1; echo "probe rc=$?"
