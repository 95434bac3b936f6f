# mbarrier try_wait suspend-time hint (exp/libkpm_hint.so, -DKPM_WAIT_HINT=20000) vs the in-tree build
mkdir -p gpurun_out/hint
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/hint/build.log 2>&1; echo "build rc=$?"
timeout 1800 python scripts/ab_libs.py --libs paper_1410_5242_b200/libkpm.so,exp/libkpm_hint.so --R 32,16,8 --rounds 3 > gpurun_out/hint/ab.jsonl 2> gpurun_out/hint/ab.err; echo "ab rc=$?"
python - <<'PY'
import json, collections
agg=collections.defaultdict(list)
for l in open("gpurun_out/hint/ab.jsonl"):
    r=json.loads(l)
    if "sweep_ms" in r: agg[(r["R"], r["lib"].split("/")[-1])].append((round(r["sweep_ms"],4), r["sm_mhz"], r["mu1"]))
    else: print(r)
for k in sorted(agg): print(k, agg[k])
PY
