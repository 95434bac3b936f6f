# Final R = 32 kernel: launch list of the bench command and ncu --set full of one main sweep
mkdir -p gpurun_out/prof4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/prof4/build.log 2>&1; echo "build rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-r-sweep --no-cpu-baseline --no-e2e"
$B > gpurun_out/prof4/bench_plain.json 2> gpurun_out/prof4/bench_plain.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/prof4/launches.csv $B > gpurun_out/prof4/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 1 -c 1 -o /tmp/full_r32 python scripts/prof_run.py --lattice 200,100,40 --M 8 --R 32 > gpurun_out/prof4/ncu_full_r32.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/full_r32.ncu-rep --page raw --csv > gpurun_out/prof4/full_r32.raw.csv 2>/dev/null
ncu -i /tmp/full_r32.ncu-rep --page source --csv --print-source sass > gpurun_out/prof4/full_r32.source.csv 2>/dev/null
