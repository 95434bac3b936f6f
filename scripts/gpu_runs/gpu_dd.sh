mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_kernel or c3 or device_build" 2>&1 | tail -2
echo short; timeout 300 python scripts/variant_sweep.py --R 32 2>&1 | grep 'tiled' | cut -c1-140
echo sustained; timeout 600 python scripts/variant_sweep.py --R 32 --M 200 --warm-seconds 4 2>&1 | grep 'tiled' | cut -c1-140
KPM_VARIANT=1 python scripts/prof_run.py --lattice 200,100,40 --R 32 --M 8 > gpurun_out/dd_plain.log 2>&1 && KPM_VARIANT=1 ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 1 -c 1 -o gpurun_out/prof_dd python scripts/prof_run.py --lattice 200,100,40 --R 32 --M 8 > /dev/null 2>&1
ls gpurun_out | grep dd
