# z-runs folded into the own copy (e32: same bytes, two copies fewer) vs dropped (e16) vs product
mkdir -p gpurun_out
for e in 0 32 16 0 32; do timeout 300 python scripts/exp_power.py $e 32 2>&1 | grep '^{'; done | tee gpurun_out/power32e.jsonl
for e in 0 32 16; do timeout 300 python scripts/exp_power.py $e 16 2>&1 | grep '^{'; done | tee gpurun_out/power16e.jsonl
