# R = 32 variants under sustained load (power cap): each variant warmed for 10 s, then timed,
# with nvidia-smi clocks sampled in the background.
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 500 > gpurun_out/sustained_clocks.csv &
SMI=$!
python scripts/variant_sweep.py --R 32 --M 400 --warm-seconds 10 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['R'], d['v'], d['kernel'], round(d['sweep_ms'],4), round(d['frac'],3), flush=True)
"
kill $SMI
