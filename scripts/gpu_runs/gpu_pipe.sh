# software-pipelined gather loop vs the defaults: full clock (short) and sustained (power cap)
mkdir -p gpurun_out
timeout 300 python scripts/variant_sweep.py --R 32 --variants 0,3,6,7,8 2>&1 | grep '^{' | tee gpurun_out/pipe_short.jsonl
timeout 300 python scripts/variant_sweep.py --R 16 --variants 0,9,10 2>&1 | grep '^{' | tee -a gpurun_out/pipe_short.jsonl
timeout 300 python scripts/variant_sweep.py --R 8 --variants 0,5 2>&1 | grep '^{' | tee -a gpurun_out/pipe_short.jsonl
timeout 600 python scripts/variant_sweep.py --R 32 --M 400 --warm-seconds 4 --variants 0,7,8,0,7 2>&1 | grep '^{' | tee gpurun_out/pipe_sust.jsonl
