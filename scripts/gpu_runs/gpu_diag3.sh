# entry-0 peel without keeping V_i (multi-CTA variants): A/B at R = 8, 16
mkdir -p gpurun_out
for e in 0 new2 0 new2; do EXP_R=8,16 timeout 300 python scripts/exp_epilogue.py $e 2>&1 | grep '^{'; done | tee gpurun_out/diag_ab3.jsonl
