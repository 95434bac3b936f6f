mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for g in 0 1; do KPM_GRAPH=$g python scripts/prof_run.py --lattice 8,8,8 --R 4 --M 64 --reps 3 | tail -1 | sed "s/^/graph=$g C1 /"; KPM_GRAPH=$g python scripts/prof_run.py --lattice 64,64,32 --R 8 --M 1000 --reps 2 | tail -1 | sed "s/^/graph=$g C2 /"; done
timeout 900 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench4.json')); print(d['value'], d['roofline'], d['cache_resident'], d['e2e'], d['clocks'])"
