# R = 32: two CTAs per SM with 1-stage rings (16 consumer warps per SM, 96 registers)
mkdir -p gpurun_out
timeout 300 python scripts/variant_sweep.py --R 32 --variants 0,6,7,8 2>&1 | grep '^{' | tee gpurun_out/m2_short.jsonl
timeout 600 python scripts/variant_sweep.py --R 32 --M 400 --warm-seconds 4 --variants 0,6,7,8,0 2>&1 | grep '^{' | tee gpurun_out/m2_sust.jsonl
