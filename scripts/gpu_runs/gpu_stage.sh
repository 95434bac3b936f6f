mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "stages or c1_all" 2>&1 | tail -2
timeout 600 python scripts/stage_ladder.py > gpurun_out/stage_ladder.json 2> gpurun_out/stage_ladder.err; echo rc=$?; cat gpurun_out/stage_ladder.json; tail -3 gpurun_out/stage_ladder.err
