# block-cache kernels: row-major index path resolved at compile time vs exp/libkpm_final.so
mkdir -p gpurun_out/ab6
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab6/build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ab6/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab6/pytest.log
timeout 1800 python scripts/ab_libs.py --libs exp/libkpm_final.so,paper_1410_5242_b200/libkpm.so --R 32,16 --rounds 3 > gpurun_out/ab6/ab.jsonl 2> gpurun_out/ab6/ab.err; echo "ab rc=$?"
python - <<'PY'
import json, collections
agg=collections.defaultdict(list)
for l in open("gpurun_out/ab6/ab.jsonl"):
    r=json.loads(l)
    if "sweep_ms" in r: agg[(r["R"], r["lib"].split("/")[-1])].append((round(r["sweep_ms"],4), r["sm_mhz"], r["mu1"]))
    else: print(r)
for k in sorted(agg): print(k, agg[k])
PY
