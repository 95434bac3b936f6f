# pair feed (race fixed): A/B timing vs tiled.bc at C3 R=32 + ncu --set full of one main sweep each
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_kernel_variant or block_cache or sell_bit or device_build" > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2b_pytest.log
timeout 600 python scripts/ab_pair.py --rounds 3 --R 32 --names tiled.bc.lpr8.u4,pair.bc.lpr8.u2,pair.bc.lpr8.u4 > gpurun_out/r2b_ab.jsonl 2> gpurun_out/r2b_ab.err; echo "ab rc=$?"
for v in tiled.bc.lpr8.u4 pair.bc.lpr8.u2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 2 -c 1 -o gpurun_out/r2b_$v python scripts/prof_run.py --R 32 --M 8 --variant $v > gpurun_out/r2b_ncu_$v.log 2>&1; echo "ncu $v rc=$?"
done
ls -la gpurun_out | tail
