# block-cache feed: parity, then sustained timing (default vs bc, storage vs y-line order)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "block_cache or c1_all or every_kernel" 2>&1 | tail -3
for cfg in "0 storage" "6 ylines" "0 ylines" "6 storage" "0 storage" "6 ylines"; do set -- $cfg
  KPM_VARIANT=$1 timeout 300 python scripts/exp_order.py $2 32 148 2>&1 | grep '^{\|rror' | tail -1; done | tee gpurun_out/bc32.jsonl
