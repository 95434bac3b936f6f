# virtual ranks with the per-sweep enqueue rendezvous (x3 repeats), then the virtual test file; strip widths 3/4 at R=32
export CUDA_DEVICE_MAX_CONNECTIONS=32
for rep in 1 2 3; do for P in 4 8; do for R in 8 32; do
  VRANKS_DUMP_AFTER=100 timeout 150 python tests/vranks_parity.py ti $P $R > gpurun_out/r2i_p${P}_r${R}_$rep.log 2>&1; echo "rep $rep P=$P R=$R rc=$? $(grep VRANKS_RESULT gpurun_out/r2i_p${P}_r${R}_$rep.log)"
done; done; done
unset CUDA_DEVICE_MAX_CONNECTIONS
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q > gpurun_out/r2i_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2i_pytest.log
for r in 0 1; do
for o in ystrips ystrips3 ystrips4; do timeout 300 python scripts/ab_variants.py --rounds 1 --R 32 --names tiled.bc.lpr8.u4 --order $o >> gpurun_out/r2i_ab.jsonl 2>> gpurun_out/r2i_ab.err; done
done
cat gpurun_out/r2i_ab.jsonl | cut -c1-200
