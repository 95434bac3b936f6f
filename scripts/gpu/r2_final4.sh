# final code on a 4-GPU box: full GPU suite (multi-rank included), Bar weak N = 1, 2, 4 (driver-like flags)
mkdir -p gpurun_out/final4
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final4/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final4/pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final4/bar_n1.json 2> gpurun_out/final4/bar_n1.err; echo "n1 rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29750 + n)) bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/final4/bar_n$n.json 2> gpurun_out/final4/bar_n$n.err; echo "n$n rc=$?"
done
python - <<'PY'
import json
for n in (1, 2, 4):
    d = json.loads(open(f"gpurun_out/final4/bar_n{n}.json").read().strip().splitlines()[-1])
    print(n, round(d["value"]), round(d["roofline"]["frac"], 4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d.get("e2e", {}).get("value"))
PY
