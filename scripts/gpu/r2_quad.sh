# Quad feed (tiled.bc.quad): parity, interleaved A/B vs the default under the power cap, ncu counters
mkdir -p gpurun_out/quad
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/quad/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "block_cache or every_kernel" > gpurun_out/quad/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/quad/pytest.log
timeout 600 python scripts/prof_run.py --R 32 --M 200 --variant tiled.bc.quad > gpurun_out/quad/prof.log 2>&1; echo "prof rc=$?"; cat gpurun_out/quad/prof.log | tail -3
timeout 1200 python scripts/ab_variants.py --R 32 --rounds 3 --names tiled.bc.lpr8.u4,tiled.bc.quad > gpurun_out/quad/ab.jsonl 2> gpurun_out/quad/ab.err; echo "ab rc=$?"
cut -c1-250 gpurun_out/quad/ab.jsonl; tail -3 gpurun_out/quad/ab.err
M="gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum"
for v in tiled.bc.lpr8.u4 tiled.bc.quad; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:aug_spmmv -s 2 -c 1 --csv python scripts/prof_run.py --R 32 --M 8 --variant $v > gpurun_out/quad/ncu_$v.csv 2>&1
done
grep -h "aug_spmmv" gpurun_out/quad/ncu_*.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | cut -c1-200
