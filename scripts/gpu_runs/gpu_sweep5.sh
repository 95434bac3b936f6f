mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for st in 1 2 3; do echo "stages=$st"; KPM_TILE_STAGES=$st timeout 300 python scripts/variant_sweep.py --R 8,16,32 2>&1 | grep tiled.lpr8 | cut -c1-150; done
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo rc=$?; cat gpurun_out/bench2.json
