o=gpurun_out/hk_configs.jsonl; : > $o
timeout 900 python bench.py --method local-hk --tau 10 --seeds 64 --steps 3 --warmup 3 --cpu-seconds 20 2>>gpurun_out/hk_configs.err | tail -1 >> $o
timeout 900 python bench.py --shape arxiv --method local-hk --tau 10 --steps 3 --warmup 3 2>>gpurun_out/hk_configs.err | tail -1 >> $o
