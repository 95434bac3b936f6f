# sanity of the other configurations with the final defaults: C2, C4 (auto order), C5 (150 GB slab)
mkdir -p gpurun_out
for c in C2 C4 C5; do timeout 1500 python bench.py --config $c --steps 3 --warmup 3 --no-r-sweep --no-cpu-baseline > gpurun_out/cfg2_$c.json 2> gpurun_out/cfg2_$c.err; echo "$c rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/cfg2_$c.json'))
print('$c', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['config']['kernel_variant'], d['config']['chunk_order'], d['config'].get('hbm_in_use_gb'))"; done
