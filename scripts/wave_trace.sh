python scripts/wave_trace.py products 1e-7 > gpurun_out/wt_products.txt 2>&1
GDIFF_WAVE_SERIAL=1 python scripts/wave_trace.py products 1e-7 > gpurun_out/wt_products_serial.txt 2>&1
python scripts/wave_trace.py papers100M 1e-6 > gpurun_out/wt_papers.txt 2>&1
GDIFF_WAVE_SERIAL=1 python scripts/wave_trace.py papers100M 1e-6 > gpurun_out/wt_papers_serial.txt 2>&1
