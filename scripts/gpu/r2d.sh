# full GPU suite (incl. virtual ranks, bench-config parity), bench with the library order, order A/B
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2d_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --chunk-order none --no-r-sweep --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench_none.json 2>> gpurun_out/r2d_bench.err; echo "bench none rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --chunk-order ylines --no-r-sweep --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench_ylines.json 2>> gpurun_out/r2d_bench.err; echo "bench ylines rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-r-sweep --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench_auto2.json 2>> gpurun_out/r2d_bench.err; echo "bench auto rc=$?"
