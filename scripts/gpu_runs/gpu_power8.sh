mkdir -p gpurun_out
for e in 0 4; do timeout 300 python scripts/exp_power.py $e 16 2>&1 | grep '^{' ; done | tee gpurun_out/power16f.jsonl
