# sustained time / SM clock / board power of the R = 32 (and 16) sweep with on-chip work removed
mkdir -p gpurun_out
for e in 0 1 2 3 0; do timeout 300 python scripts/exp_power.py $e 32 2>&1 | grep '^{'; done | tee gpurun_out/power32.jsonl
for e in 0 1 3; do timeout 300 python scripts/exp_power.py $e 16 2>&1 | grep '^{'; done | tee gpurun_out/power16.jsonl
