# L2 policy of the streamed W / val / lcol copies and the W stores, sustained power / clock
mkdir -p gpurun_out
for p in 0 1 2 0 1 2; do KPM_STREAM_POLICY=$p timeout 300 python scripts/exp_order.py storage 32 148 2>&1 | grep '^{' | sed "s/^{/{\"policy\": $p, /"; done | tee gpurun_out/policy32.jsonl
for p in 0 1 2; do KPM_STREAM_POLICY=$p timeout 300 python scripts/exp_order.py storage 16 296 2>&1 | grep '^{' | sed "s/^{/{\"policy\": $p, /"; done | tee gpurun_out/policy16.jsonl
