timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "every_kernel_variant" > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2u_pytest.log
timeout 900 python scripts/ab_variants.py --rounds 3 --R 8 --names tiled.lpr4.u4.wr.s2,tiled.lpr2.u4.wr.s2,tiled.bc.lpr2.u4.wr,tiled.bc.lpr4.u4.wr > gpurun_out/r2u_ab.jsonl 2> gpurun_out/r2u_ab.err; echo "ab rc=$?"
cut -c1-170 gpurun_out/r2u_ab.jsonl
