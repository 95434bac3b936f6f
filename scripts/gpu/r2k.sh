# R=32 block-cache feed with W in registers vs W staged (3 rounds, library order)
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "every_kernel_variant" > gpurun_out/r2k_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2k_pytest.log
timeout 900 python scripts/ab_variants.py --rounds 4 --R 32 --names tiled.bc.lpr8.u4,tiled.bc.lpr8.u4.wr > gpurun_out/r2k_ab.jsonl 2> gpurun_out/r2k_ab.err; echo "ab rc=$?"
cat gpurun_out/r2k_ab.jsonl | cut -c1-160
