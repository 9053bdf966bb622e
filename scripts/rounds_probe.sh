for off in 0 512; do
python scripts/rounds_probe.py products 1e-7 $off > gpurun_out/rp_base_$off.txt 2>&1
GDIFF_GROUP_MIN=0 python scripts/rounds_probe.py products 1e-7 $off > gpurun_out/rp_g0_$off.txt 2>&1
GDIFF_GROUP_MIN=0 GDIFF_SLOT_GROUP=64 python scripts/rounds_probe.py products 1e-7 $off > gpurun_out/rp_g0s64_$off.txt 2>&1
GDIFF_GROUP_MIN=0 GDIFF_SLOT_GROUP=1 python scripts/rounds_probe.py products 1e-7 $off > gpurun_out/rp_g0s1_$off.txt 2>&1
done
