mkdir -p gpurun_out
nproc; free -g | head -2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo rc=$?; cat gpurun_out/bench3.json
