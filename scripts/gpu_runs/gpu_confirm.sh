# Round-end style confirmation on one B200: GPU test suite, smoke(), default bench line.
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/confirm_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/confirm_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/confirm_bench.json 2> gpurun_out/confirm_bench.err; echo "bench rc=$?"
cut -c1-400 gpurun_out/confirm_bench.json
