timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2o_bench.json 2> gpurun_out/r2o_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-r-sweep > gpurun_out/r2o_c1.json 2>> gpurun_out/r2o_bench.err; echo "c1 rc=$?"
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-r-sweep > gpurun_out/r2o_c2.json 2>> gpurun_out/r2o_bench.err; echo "c2 rc=$?"
python - <<'PY'
import json
for f in ("r2o_bench","r2o_c1","r2o_c2"):
    d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, round(d["value"]), d["roofline"]["frac"], d.get("cache_roofline"), d["clocks"]["sm_mhz"], d["run"]["kernel_variant"])
PY
