# block-cache feed at R = 32 and 16: parity, then sustained timing (default vs bc with the y-line order)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "block_cache or every_kernel or c1_all" 2>&1 | tail -3
for cfg in "0 storage 32 148" "6 ylines 32 148" "0 storage 16 296" "1 ylines 16 296" "0 storage 32 148" "6 ylines 32 148" "0 storage 16 296" "1 ylines 16 296"; do set -- $cfg
  KPM_VARIANT=$1 timeout 300 python scripts/exp_order.py $2 $3 $4 2>&1 | grep '^{\|rror' | tail -1; done | tee gpurun_out/bc2.jsonl
