# single-group row-pair feed vs tiled.bc at C3 R=32: parity of every variant, A/B, ncu of the pair kernel
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_kernel_variant or sell_bit or device_build or c3_sampled" > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2c_pytest.log
timeout 600 python scripts/ab_pair.py --rounds 3 --R 32 --names tiled.bc.lpr8.u4,pair.bc.lpr8.u2,pair.bc.lpr8.u4,pair.bc.lpr8.u4.v2 > gpurun_out/r2c_ab.jsonl 2> gpurun_out/r2c_ab.err; echo "ab rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 2 -c 1 -o gpurun_out/r2c_pair python scripts/prof_run.py --R 32 --M 8 --variant pair.bc.lpr8.u4 > gpurun_out/r2c_ncu.log 2>&1; echo "ncu rc=$?"
