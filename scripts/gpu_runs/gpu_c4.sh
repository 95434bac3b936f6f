mkdir -p gpurun_out
for c in C1 C2 C4; do
timeout 900 python bench.py --config $c --no-cpu-baseline --no-r-sweep > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', d['value'], d['roofline']['sweep_ms'], d['roofline']['frac'], d['roofline']['traffic'], d['e2e']['value'], d['clocks'])"
done
python scripts/prof_run.py --lattice 400,400,40 --R 32 --M 8 > gpurun_out/p_c4.log 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:aug_spmmv -s 1 -c 2 python scripts/prof_run.py --lattice 400,400,40 --R 32 --M 8 > gpurun_out/ncu_c4.txt 2>&1
grep -E "dram__bytes|duration|wavefronts|hit_rate" gpurun_out/ncu_c4.txt
