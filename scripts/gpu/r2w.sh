# validate the row-major tile indices default: full GPU suite (2 GPUs), bench, ncu of R = 32 / 16
mkdir -p gpurun_out/prof3
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/prof3/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/prof3/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/prof3/bench.json 2> gpurun_out/prof3/bench.err; echo "bench rc=$?"
P="python scripts/prof_run.py --lattice 200,100,40 --M 8"
for r in 32 16; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 1 -c 1 -o /tmp/full_r$r $P --R $r > gpurun_out/prof3/ncu_full_r$r.log 2>&1; echo "ncu R=$r rc=$?"
  ncu -i /tmp/full_r$r.ncu-rep --page raw --csv > gpurun_out/prof3/full_r$r.raw.csv 2>/dev/null
done
cp /tmp/full_r32.ncu-rep gpurun_out/prof3/
python - <<'PY'
import json
d=json.loads(open("gpurun_out/prof3/bench.json").read().strip().splitlines()[-1])
print(round(d["value"]), d["roofline"]["frac"], d["clocks"]["sm_mhz"], {k:round(v["frac"],3) for k,v in d["by_R"].items()})
PY
