# incremental ring counters (no runtime division per tile): full GPU suite, then A/B vs the previous build
mkdir -p gpurun_out/abdiv
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/abdiv/build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/abdiv/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/abdiv/pytest.log
timeout 1800 python scripts/ab_libs.py --libs exp/libkpm_old.so,paper_1410_5242_b200/libkpm.so --R 32,16,8,4,1 --rounds 3 > gpurun_out/abdiv/ab.jsonl 2> gpurun_out/abdiv/ab.err; echo "ab rc=$?"
python - <<'PY'
import json, collections
rows=[json.loads(l) for l in open("gpurun_out/abdiv/ab.jsonl") if l.strip()]
agg=collections.defaultdict(list)
for r in rows:
    if "sweep_ms" in r: agg[(r["R"], r["lib"].split("/")[-1])].append((r["sweep_ms"], r["sm_mhz"], r["frac"]))
for k in sorted(agg): print(k, [round(x[0],4) for x in agg[k]], [x[1] for x in agg[k]], round(sum(x[2] for x in agg[k])/len(agg[k]),4))
PY
