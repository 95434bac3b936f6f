mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "block_cache or every_kernel or c1_all" > gpurun_out/bc3.log 2>&1; tail -40 gpurun_out/bc3.log | cut -c1-300
