# final state check on one B200: GPU test suite, smoke(), default bench line, then the R=16 power repeat
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/confirm2_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/confirm2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/confirm2_bench.json 2> gpurun_out/confirm2_bench.err; echo "bench rc=$?"
cut -c1-200 gpurun_out/confirm2_bench.json
bash scripts/gpu_runs/gpu_power3.sh
