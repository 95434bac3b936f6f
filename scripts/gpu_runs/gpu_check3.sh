mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "every_kernel or c1_all" 2>&1 | tail -3
timeout 600 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python scripts/prof_run.py --lattice 6,5,9 --R 1,4,8,16,32 --M 16 > gpurun_out/memcheck.log 2>&1; echo memcheck rc=$?
tail -5 gpurun_out/memcheck.log
