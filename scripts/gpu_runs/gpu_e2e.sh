mkdir -p gpurun_out
for st in 2 3 5; do
python bench.py --steps $st --warmup 3 --no-r-sweep --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']
print('steps', d['steps'], 'dev ms', round(d['ms_per_step'],1), 'e2e ms', round(e['ms_per_step'],1), 'set_matrix ms', round(e['set_matrix_ms_per_step'],1), 'clk', d['clocks']['sm_mhz'])"
done
python scripts/time_e2e.py
