timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "block_cache or full_m_r16" > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2q_pytest.log
