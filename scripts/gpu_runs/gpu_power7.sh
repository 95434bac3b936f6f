mkdir -p gpurun_out
for e in 0 16 8 4 1; do timeout 300 python scripts/exp_power.py $e 32 2>&1 | grep '^{\|Error' | tail -2; done | tee gpurun_out/power32f.jsonl
