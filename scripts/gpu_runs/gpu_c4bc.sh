# C4 (400x400x40, 1 GPU): y-band order (auto) vs y-line walks with the block cache
mkdir -p gpurun_out
for o in auto ylines; do
  timeout 900 python bench.py --config C4 --chunk-order $o --steps 3 --warmup 3 --no-r-sweep --no-cpu-baseline --no-e2e > gpurun_out/c4_$o.json 2> gpurun_out/c4_$o.err; echo "$o rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/c4_$o.json'))
print('$o', round(d['value']), round(d['roofline']['frac'],3), d['roofline']['sweep_ms'], d['clocks']['sm_mhz'], d['config']['kernel_variant'], d['config']['chunk_order'])"
done
