# block cache as the R = 16 / 32 default: GPU test suite, smoke, default bench line
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/bc4_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/bc4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bc4_bench.json 2> gpurun_out/bc4_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bc4_bench.err
python -c "
import json; d=json.load(open('gpurun_out/bc4_bench.json'))
print(d['value'], d['roofline']['frac'], d['roofline']['sweep_ms'], d['clocks'], d['config']['kernel_variant'], d['config']['chunk_order'], d['e2e']['value'])
print({R:(round(v['frac'],3), v['kernel']) for R,v in d['by_R'].items()})"
