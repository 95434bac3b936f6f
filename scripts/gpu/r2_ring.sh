# deeper block-cache rings (old W via registers): parity, interleaved A/B vs the defaults
mkdir -p gpurun_out/ring
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ring/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "block_cache or every_kernel" > gpurun_out/ring/pytest.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/ring/pytest.log
timeout 1500 python scripts/ab_variants.py --R 32 --rounds 3 --names tiled.bc.lpr8.u4,tiled.bc.lpr8.u4.wr.s3,tiled.bc.lpr8.u4.wr.s4,tiled.bc.lpr8.u4.s3 > gpurun_out/ring/ab32.jsonl 2> gpurun_out/ring/ab32.err; echo "ab32 rc=$?"
timeout 900 python scripts/ab_variants.py --R 16 --rounds 3 --names tiled.bc.lpr8.u4.wr,tiled.bc.lpr8.u4.wr.s3 > gpurun_out/ring/ab16.jsonl 2> gpurun_out/ring/ab16.err; echo "ab16 rc=$?"
python - <<'PY'
import json, collections
for f in ("ab32", "ab16"):
    agg=collections.defaultdict(list)
    for l in open(f"gpurun_out/ring/{f}.jsonl"):
        r=json.loads(l); agg[(r["R"], r["variant"], r["ran"])].append((round(r["sweep_ms"],4), r.get("sm_mhz")))
    for k in agg: print(k, agg[k])
PY
