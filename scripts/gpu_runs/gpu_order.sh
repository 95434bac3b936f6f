mkdir -p gpurun_out
for m in storage zcol storage zcol; do timeout 300 python scripts/exp_order.py $m 32 148 2>&1 | grep '^{'; done | tee gpurun_out/order32.jsonl
for m in storage zcol; do timeout 300 python scripts/exp_order.py $m 16 296 2>&1 | grep '^{'; done | tee gpurun_out/order16.jsonl
