# lcol-preload variants vs defaults (library order), 3 rounds; ncu of the R=32 preload kernel
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "every_kernel_variant" > gpurun_out/r2j_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2j_pytest.log
timeout 900 python scripts/ab_variants.py --rounds 3 --R 32,16 --names tiled.bc.lpr8.u4,tiled.bc.lpr8.u4.pl,tiled.bc.lpr8.u4.wr,tiled.bc.lpr8.u4.wr.pl > gpurun_out/r2j_ab.jsonl 2> gpurun_out/r2j_ab.err; echo "ab rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 2 -c 1 -o gpurun_out/r2j_pl python scripts/prof_run.py --R 32 --M 8 --variant tiled.bc.lpr8.u4.pl > gpurun_out/r2j_ncu.log 2>&1; echo "ncu rc=$?"
