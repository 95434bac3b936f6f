# which copies cost the clock: x+-1 blocks (e8), z-runs (e16), y+-1 (e4), all non-own (e1)
mkdir -p gpurun_out
for e in 0 8 16 4 1 0 8 16; do timeout 300 python scripts/exp_power.py $e 32 2>&1 | grep '^{'; done | tee gpurun_out/power32d.jsonl
for e in 0 8 16; do timeout 300 python scripts/exp_power.py $e 16 2>&1 | grep '^{'; done | tee gpurun_out/power16d.jsonl
