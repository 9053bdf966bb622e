bash scripts/ab.sh ab_bal.txt "--steps 20 --warmup 3" "--eps 1e-6 --steps 20 --warmup 3" "--shape papers100M --eps 1e-6 --steps 5 --warmup 3" "--shape papers100M --eps 1e-7 --steps 5 --warmup 3"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gputests_bal.log 2>&1; tail -3 gpurun_out/gputests_bal.log
