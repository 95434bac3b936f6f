# A/B of the working tree's libkpm.so against exp/libkpm_head.so (the last commit): GPU parity suite,
# interleaved timing, ncu instruction / wavefront counts of one R = 32 sweep for each
mkdir -p gpurun_out/ab2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab2/build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ab2/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab2/pytest.log
timeout 1800 python scripts/ab_libs.py --libs exp/libkpm_head.so,paper_1410_5242_b200/libkpm.so --R ${ABR:-32,16,8,4} --rounds 3 > gpurun_out/ab2/ab.jsonl 2> gpurun_out/ab2/ab.err; echo "ab rc=$?"
python - <<'PY'
import json, collections
rows=[json.loads(l) for l in open("gpurun_out/ab2/ab.jsonl") if l.strip()]
agg=collections.defaultdict(list)
for r in rows:
    if "sweep_ms" in r: agg[(r["R"], r["lib"].split("/")[-1])].append((r["sweep_ms"], r["sm_mhz"], r["frac"]))
    else: print(r)
for k in sorted(agg): print(k, [round(x[0],4) for x in agg[k]], [x[1] for x in agg[k]], round(sum(x[2] for x in agg[k])/len(agg[k]),4))
PY
M="gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active"
for L in exp/libkpm_head.so paper_1410_5242_b200/libkpm.so; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:aug_spmmv -s 2 -c 1 --csv python -c "
import sys; sys.argv=['x','--R','32','--M','8']; sys.path.insert(0,'.'); sys.path.insert(0,'scripts')
import paper_1410_5242_b200 as k; k.LIB_PATH='$L'
import prof_run; prof_run.main()" > gpurun_out/ab2/ncu_$(basename $L).csv 2>&1
  grep -h "aug_spmmv" gpurun_out/ab2/ncu_$(basename $L).csv | awk -F'","' '{print "'$(basename $L)'", $(NF-2), $NF}'
done
