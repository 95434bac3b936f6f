# virtual ranks after the kernel preload fix (x3 repeats of the formerly hanging cases), then the full GPU suite
export VRANKS_TRACE=1
for rep in 1 2 3; do for P in 4 8; do for R in 8 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=32 VRANKS_DUMP_AFTER=100 timeout 150 python tests/vranks_parity.py ti $P $R > gpurun_out/r2g_p${P}_r${R}_$rep.log 2>&1; echo "rep $rep P=$P R=$R rc=$? $(grep VRANKS_RESULT gpurun_out/r2g_p${P}_r${R}_$rep.log)"
done; done; done
unset VRANKS_TRACE
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2g_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
