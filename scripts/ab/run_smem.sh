# shared-memory CTA form: GPU tests of the batch paths + cora / config-1 A/B
timeout 1500 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/smem_tests.log 2>&1; tail -3 gpurun_out/smem_tests.log
o=gpurun_out/smem_ab.txt; : > $o
for env in "GDIFF_CTA_SMEM=0" "X=1"; do
  env $env timeout 600 python bench.py --shape cora --eps 1e-6 --seeds 50 --steps 20 --warmup 3 --no-cpu-baseline 2>>$o.err | tail -1 | sed "s|^|$env [cora 50] |" >> $o
  env $env timeout 600 python bench.py --shape cora --eps 1e-6 --seeds 1024 --steps 10 --warmup 3 --no-cpu-baseline 2>>$o.err | tail -1 | sed "s|^|$env [cora 1024] |" >> $o
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_seed_smem" -s 5 -c 1 -o gpurun_out/prof_k_seed_smem_r02 python bench.py --shape cora --eps 1e-6 --seeds 50 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_smem.log 2>&1; echo "ncu rc=$?"
