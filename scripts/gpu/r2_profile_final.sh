# Final round-2 profiles: launch list of the bench command, ncu --set full of the main sweep per R
# (raw CSV exports; the R = 32 report and its SASS source counters kept)
mkdir -p gpurun_out/prof3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/prof3/build.log 2>&1; echo "build rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-r-sweep --no-cpu-baseline --no-e2e"
$B > gpurun_out/prof3/bench_plain.json 2> gpurun_out/prof3/bench_plain.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/prof3/launches.csv $B > gpurun_out/prof3/ncu_launch.log 2>&1; echo "launch list rc=$?"
P="python scripts/prof_run.py --lattice 200,100,40 --M 8"
for r in 32 16 8 4 2 1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 1 -c 1 -o /tmp/full_r$r $P --R $r > gpurun_out/prof3/ncu_full_r$r.log 2>&1; echo "ncu R=$r rc=$?"
  ncu -i /tmp/full_r$r.ncu-rep --page raw --csv > gpurun_out/prof3/full_r$r.raw.csv 2>/dev/null
done
ncu -i /tmp/full_r32.ncu-rep --page source --csv --print-source sass > gpurun_out/prof3/full_r32.source.csv 2>/dev/null
cp /tmp/full_r32.ncu-rep gpurun_out/prof3/
du -sh gpurun_out
