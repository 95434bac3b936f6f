mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
echo "short"; timeout 300 python scripts/variant_sweep.py --R 1,2,4,16 2>&1 | cut -c1-150
for st in 1 3 4; do echo "stages=$st"; KPM_TILE_STAGES=$st timeout 300 python scripts/variant_sweep.py --R 1,2,4 2>&1 | grep tiled | cut -c1-150; done
