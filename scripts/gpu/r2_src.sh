# ncu --set full with SASS source counters of the R = 32 default sweep (instruction mix per line)
mkdir -p gpurun_out/src
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/src/build.log 2>&1; echo "build rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:aug_spmmv -s 2 -c 1 -o gpurun_out/src/r32 python scripts/prof_run.py --R 32 --M 8 > gpurun_out/src/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/src/r32.ncu-rep --page source --csv --print-source sass > gpurun_out/src/r32_sass.csv 2>&1; echo "export rc=$?"
ls -la gpurun_out/src
