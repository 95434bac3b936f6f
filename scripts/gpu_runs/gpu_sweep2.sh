mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 600 python scripts/variant_sweep.py --R 8,16,32 2>&1 | tee gpurun_out/variants2.jsonl | cut -c1-200
for st in 2 3; do echo "stages=$st"; KPM_TILE_STAGES=$st timeout 300 python scripts/variant_sweep.py --R 8,16,32 2>&1 | grep tiled | cut -c1-200; done
