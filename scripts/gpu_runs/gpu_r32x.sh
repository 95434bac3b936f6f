# R = 32 lane-map experiments: full clock (short) and sustained (power cap) sweeps of every variant
mkdir -p gpurun_out
timeout 600 python scripts/variant_sweep.py --R 32 2>&1 | grep '^{' | tee gpurun_out/r32x_short.jsonl
timeout 900 python scripts/variant_sweep.py --R 32 --M 400 --warm-seconds 4 --variants 0,6,7,8,9,10,11 2>&1 | grep '^{' | tee gpurun_out/r32x_sust.jsonl
