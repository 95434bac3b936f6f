# sustained: product vs "no y+-1 block copies" (e4, what a block cache would save) vs no non-own copies (e1)
mkdir -p gpurun_out
for e in 0 4 1 0 4; do timeout 300 python scripts/exp_power.py $e 32 2>&1 | grep '^{'; done | tee gpurun_out/power32b.jsonl
for e in 0 4 1; do timeout 300 python scripts/exp_power.py $e 16 2>&1 | grep '^{'; done | tee gpurun_out/power16b.jsonl
