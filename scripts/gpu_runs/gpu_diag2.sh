# own-row-first SELL order (peel only without a multi-CTA register cap): A/B at every width
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for e in 0 new 0 new; do EXP_R=1,2,4,8,16,32 timeout 300 python scripts/exp_epilogue.py $e 2>&1 | grep '^{'; done | tee gpurun_out/diag_ab2.jsonl
