# own-row-first SELL order: GPU tests, then A/B sweep timing against the previous library
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for e in 0 new 0 new; do timeout 300 python scripts/exp_epilogue.py $e 2>&1 | grep '^{'; done | tee gpurun_out/diag_ab.jsonl
