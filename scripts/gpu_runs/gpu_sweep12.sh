mkdir -p gpurun_out
for st in 2 3; do echo "stages=$st"; KPM_TILE_STAGES=$st timeout 300 python scripts/variant_sweep.py --R 8,16,32 2>&1 | grep 'tiled.lpr8.u4' | cut -c1-120; done
echo "sustained stages=2"; KPM_TILE_STAGES=2 timeout 600 python scripts/variant_sweep.py --R 16 --M 200 --warm-seconds 4 2>&1 | grep 'tiled.lpr8.u4' | cut -c1-120
echo "sustained stages=3"; KPM_TILE_STAGES=3 timeout 600 python scripts/variant_sweep.py --R 16 --M 200 --warm-seconds 4 2>&1 | grep 'tiled.lpr8.u4' | cut -c1-120
