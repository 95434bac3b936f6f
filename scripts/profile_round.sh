# Profiles for profiles/: launch list of the bench command + ncu --set full of the hot kernel per R.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-r-sweep --no-cpu-baseline"
$B > gpurun_out/prof_bench_plain.json 2> gpurun_out/prof_bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
P="python scripts/prof_run.py --lattice 200,100,40 --M 8"
$P --R 32,16,8,4,2,1 > gpurun_out/prof_plain.log 2>&1 || exit 1
for r in 32 16 8 4 2 1; do
  ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 1 -c 1 -o gpurun_out/full_r$r $P --R $r > gpurun_out/ncu_full_r$r.log 2>&1
done
ls -la gpurun_out
