mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 900 python scripts/variant_sweep.py --grid-per-sm 0,1,2,3 2>&1 | tee gpurun_out/variants.jsonl | tail -80
