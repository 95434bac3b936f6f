timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "degenerate or fig1 or z4 or timing" > gpurun_out/r2m_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2m_pytest.log
