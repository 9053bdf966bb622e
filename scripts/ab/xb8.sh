bash scripts/ab.sh ab_xb8.txt "--steps 20 --warmup 3" "--eps 1e-6 --steps 20 --warmup 3"
