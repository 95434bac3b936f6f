# block cache at R = 8: parity, then sustained A/B (base variant, storage order vs block cache, y-lines)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "block_cache or every_kernel or c1_all" 2>&1 | tail -2
for cfg in "1 storage 8 444" "0 ylines 8 444" "1 storage 8 444" "0 ylines 8 444"; do set -- $cfg
  KPM_VARIANT=$1 timeout 300 python scripts/exp_order.py $2 $3 $4 2>&1 | grep '^{\|rror' | tail -1; done | tee gpurun_out/bc8.jsonl
