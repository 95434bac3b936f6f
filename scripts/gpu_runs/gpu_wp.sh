# old W prefetched one tile ahead (wp) vs the defaults: short (full clock) and sustained
mkdir -p gpurun_out
timeout 300 python scripts/variant_sweep.py --R 32 --variants 0,1,6,7 2>&1 | grep '^{' | tee gpurun_out/wp_short.jsonl
timeout 300 python scripts/variant_sweep.py --R 16 --variants 0,9 2>&1 | grep '^{' | tee -a gpurun_out/wp_short.jsonl
timeout 300 python scripts/variant_sweep.py --R 8 --variants 0,5 2>&1 | grep '^{' | tee -a gpurun_out/wp_short.jsonl
timeout 600 python scripts/variant_sweep.py --R 32 --M 400 --warm-seconds 4 --variants 0,6,7,0,6 2>&1 | grep '^{' | tee gpurun_out/wp_sust.jsonl
timeout 600 python scripts/variant_sweep.py --R 16 --M 400 --warm-seconds 4 --variants 0,9,0,9 2>&1 | grep '^{' | tee -a gpurun_out/wp_sust.jsonl
