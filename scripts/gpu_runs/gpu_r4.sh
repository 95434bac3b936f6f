mkdir -p gpurun_out
python scripts/variant_sweep.py --R 4,16 --M 200 --grid-per-sm 0 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['R'], d['v'], d['grid_per_sm'], d['kernel'], round(d['sweep_ms'],4), round(d['frac'],3))
"
