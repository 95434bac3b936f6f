# C4 strong and C5 weak with the final kernels on a 4-GPU box (NCCL INIT lines on stderr)
mkdir -p gpurun_out/scalef
run() { local n=$1; shift; local tag=$1; shift
  if [ "$n" = 1 ]; then timeout 1200 python bench.py --gpus 1 "$@" > gpurun_out/scalef/${tag}_n1.json 2> gpurun_out/scalef/${tag}_n1.err
  else timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800 + n)) bench.py --gpus $n "$@" > gpurun_out/scalef/${tag}_n$n.json 2> gpurun_out/scalef/${tag}_n$n.err; fi
  echo "$tag n=$n rc=$? $(tail -c 200 gpurun_out/scalef/${tag}_n$n.json | head -c 0)"; }
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/scalef/build.log 2>&1
for n in 1 2 4; do run $n c4 --config C4 --steps 3 --warmup 3 --no-r-sweep --no-cpu-baseline --no-e2e; done
run 1 c5 --config C5 --steps 2 --warmup 3 --no-r-sweep --no-cpu-baseline --no-e2e
run 4 c5 --config C5 --steps 2 --warmup 3 --no-r-sweep --no-cpu-baseline --no-e2e
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/scalef/*_n*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], round(d["value"]), round(d["roofline"]["frac"], 4), d["clocks"]["sm_mhz"], d["config"]["workload"])
    except Exception as e:
        print(f, "ERR", e)
PY
