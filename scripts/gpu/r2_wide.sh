# block-cache parity on wider rows (tests/test_gpu_parity.py::test_block_cache_wide_rows)
mkdir -p gpurun_out/wide
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/wide/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "wide_rows or block_cache_feed" > gpurun_out/wide/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/wide/pytest.log
