# Round-2 profiles with the final defaults: launch list of the bench command, ncu --set full of the
# main sweep per R (library chunk order; raw CSV exports, only the R = 32 report kept), then the A/B
# of the split-accumulator variants.
mkdir -p gpurun_out/prof2
B="python bench.py --steps 2 --warmup 3 --no-r-sweep --no-cpu-baseline --no-e2e"
$B > gpurun_out/prof2/bench_plain.json 2> gpurun_out/prof2/bench_plain.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/prof2/launches.csv $B > gpurun_out/prof2/ncu_launch.log 2>&1; echo "launch list rc=$?"
P="python scripts/prof_run.py --lattice 200,100,40 --M 8"
for r in 32 16 8 4 2 1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 1 -c 1 -o /tmp/full_r$r $P --R $r > gpurun_out/prof2/ncu_full_r$r.log 2>&1; echo "ncu R=$r rc=$?"
  ncu -i /tmp/full_r$r.ncu-rep --page raw --csv > gpurun_out/prof2/full_r$r.raw.csv 2>/dev/null
done
ncu -i /tmp/full_r32.ncu-rep --page source --csv --print-source sass > gpurun_out/prof2/full_r32.source.csv 2>/dev/null
cp /tmp/full_r32.ncu-rep gpurun_out/prof2/
timeout 900 python scripts/ab_variants.py --rounds 3 --R 32,16 --names tiled.bc.lpr8.u4,tiled.bc.lpr8.u4.a2,tiled.bc.lpr8.u4.wr,tiled.bc.lpr8.u4.wr.a2 > gpurun_out/prof2/ab_a2.jsonl 2> gpurun_out/prof2/ab_a2.err; echo "ab rc=$?"
du -sh gpurun_out
