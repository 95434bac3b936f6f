mkdir -p gpurun_out
CMD="python scripts/prof_run.py --lattice 200,100,40 --R 32,8 --M 8"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:aug_spmmv_kernel -s 1 -c 1 -o gpurun_out/prof_r32 python scripts/prof_run.py --lattice 200,100,40 --R 32 --M 8 > gpurun_out/ncu_r32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:aug_spmmv_kernel -s 1 -c 1 -o gpurun_out/prof_r8 python scripts/prof_run.py --lattice 200,100,40 --R 8 --M 8 > gpurun_out/ncu_r8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:aug_spmmv_kernel -s 1 -c 1 -o gpurun_out/prof_r1 python scripts/prof_run.py --lattice 200,100,40 --R 1 --M 8 > gpurun_out/ncu_r1.log 2>&1
for s in 4 16 64; do KPM_SEGMENT=$s python scripts/prof_run.py --lattice 200,100,40 --R 32,16,8 --M 40 --reps 2 >> gpurun_out/seg.log 2>&1; echo "seg $s" >> gpurun_out/seg.log; done
for g in 1 2; do for s in 1 16 64; do KPM_GRID_PER_SM=$g KPM_SEGMENT=$s python scripts/prof_run.py --lattice 200,100,40 --R 32,16 --M 40 --reps 2 >> gpurun_out/seg.log 2>&1; echo "grid/sm $g seg $s" >> gpurun_out/seg.log; done; done
cat gpurun_out/prof_plain.log gpurun_out/seg.log
