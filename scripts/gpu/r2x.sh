# R = 32 block-cache feed with the column split (16 consumer warps), A/B vs the default; DFMA peak
mkdir -p gpurun_out/r2x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_dfma scripts/mb_dfma.cu && /tmp/mb_dfma > gpurun_out/r2x/dfma.json; cat gpurun_out/r2x/dfma.json
timeout 900 python scripts/ab_variants.py --R 32 --rounds 3 --names tiled.bc.lpr8.u4,tiled.bc.lpr8.u4.cs2,tiled.bc.lpr8.u2.cs2 > gpurun_out/r2x/ab.jsonl 2> gpurun_out/r2x/ab.err; echo "ab rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r2x/ab.jsonl"):
    d=json.loads(l); print(d["round"], d["variant"], d["ran"], round(d["sweep_ms"],4), round(d["frac"],3), d["dmu"], d["sm_mhz"], d["power_w"])
PY
P="python scripts/prof_run.py --lattice 200,100,40 --M 8"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:aug_spmmv -s 1 -c 1 -o /tmp/cs2 $P --R 32 --variant tiled.bc.lpr8.u4.cs2 > gpurun_out/r2x/ncu_cs2.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/cs2.ncu-rep --page raw --csv > gpurun_out/r2x/cs2.raw.csv 2>/dev/null
