# virtual ranks (subprocess, CUDA_DEVICE_MAX_CONNECTIONS=32), R=16/8 default candidates, y-strip order, by_R
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q > gpurun_out/r2e_pytest.log 2>&1; echo "virtual rc=$?"; tail -3 gpurun_out/r2e_pytest.log
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "every_kernel_variant or block_cache" > gpurun_out/r2e_pytest2.log 2>&1; echo "variants rc=$?"; tail -2 gpurun_out/r2e_pytest2.log
for r in 0 1; do
timeout 600 python scripts/ab_variants.py --rounds 1 --R 16 --names tiled.bc.lpr4.u4.wr,tiled.bc.lpr8.u4.wr,tiled.lpr8.u4.wr.s2,tiled.lpr4.u4.wr.s2 >> gpurun_out/r2e_ab.jsonl 2>> gpurun_out/r2e_ab.err
timeout 600 python scripts/ab_variants.py --rounds 1 --R 8 --names tiled.lpr4.u4.wr.s2,tiled.bc.lpr4.u4.wr >> gpurun_out/r2e_ab.jsonl 2>> gpurun_out/r2e_ab.err
timeout 600 python scripts/ab_variants.py --rounds 1 --R 32,16 --names tiled.bc.lpr8.u4,tiled.bc.lpr4.u4.wr,tiled.bc.lpr8.u4.wr --order ystrips >> gpurun_out/r2e_ab.jsonl 2>> gpurun_out/r2e_ab.err
timeout 600 python scripts/ab_variants.py --rounds 1 --R 32 --names tiled.bc.lpr8.u4 >> gpurun_out/r2e_ab.jsonl 2>> gpurun_out/r2e_ab.err
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo "bench rc=$?"
