# ncu --set full with source-level (SASS) stall sampling of the R = 32 main sweep
mkdir -p gpurun_out
P="python scripts/prof_run.py --lattice 200,100,40 --M 8 --R 32"
$P > gpurun_out/src32_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 2 -c 1 -o gpurun_out/src32 $P > gpurun_out/src32_ncu.log 2>&1
ncu -i gpurun_out/src32.ncu-rep --page source --csv --print-source sass > gpurun_out/src32_sass.csv 2>&1
ls -la gpurun_out/src32*
