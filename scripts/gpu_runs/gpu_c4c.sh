mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "chunk_order or c1_all" 2>&1 | tail -2
timeout 900 python bench.py --config C4 --no-cpu-baseline --no-r-sweep --no-e2e > gpurun_out/bench_C4o.json 2> gpurun_out/bench_C4o.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_C4o.json')); print(d['value'], d['roofline']['sweep_ms'], d['roofline']['frac'], d['config']['chunk_order'], d['clocks'])"
tail -3 gpurun_out/bench_C4o.err
