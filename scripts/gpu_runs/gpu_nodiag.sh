timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rows_without_diagonal or device_build or sell_bit_exact" 2>&1 | tail -15
