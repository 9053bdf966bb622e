cd "$(dirname "$0")/.."
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_wave_extract|k_wave_reset" -s 40 -c 2 \
  -o gpurun_out/prof_extract_r02 python scripts/wave_trace.py products 1e-7 > gpurun_out/ncu_extract.log 2>&1; echo "rc=$?"
