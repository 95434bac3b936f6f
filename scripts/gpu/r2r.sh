timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r2r_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2r_pytest.log
