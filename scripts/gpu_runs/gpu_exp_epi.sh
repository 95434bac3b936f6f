# exp_epilogue.py: sweep time with parts of the epilogue / index traffic removed (timing only)
mkdir -p gpurun_out
for e in 0 4 8 12 16 28 0; do timeout 300 python scripts/exp_epilogue.py $e 2>&1 | grep '^{'; done | tee gpurun_out/exp_epi.jsonl
