mkdir -p gpurun_out
P="python scripts/prof_run.py --lattice 200,100,40 --M 8"
$P --R 32 > gpurun_out/p2_plain.log 2>&1 || exit 1
KPM_VARIANT=4 ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 1 -c 1 -o gpurun_out/prof_staged32 $P --R 32 > /dev/null 2>&1
KPM_VARIANT=0 ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 1 -c 1 -o gpurun_out/prof_tiled32 $P --R 32 > /dev/null 2>&1
KPM_TILE_STAGES=2 KPM_VARIANT=0 ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 1 -c 1 -o gpurun_out/prof_tiled8 $P --R 8 > /dev/null 2>&1
ls -la gpurun_out
