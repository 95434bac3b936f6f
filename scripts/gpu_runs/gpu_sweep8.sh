mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
echo "short"; timeout 300 python scripts/variant_sweep.py --R 8,16,32 2>&1 | grep 'tiled' | cut -c1-150
echo "sustained"; timeout 600 python scripts/variant_sweep.py --R 8,16,32 --M 200 --warm-seconds 4 2>&1 | grep 'tiled.lpr8.u4"' | cut -c1-150
