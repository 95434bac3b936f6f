# profiles after the block-cache default: capture, summarise on the box (profiles/ copied into
# gpurun_out/prof_new/), keep only the R = 32 report so the results fit the 64 MiB return
bash scripts/profile_round.sh > /dev/null 2>&1
python scripts/ncu_summary.py --round r01 --launches gpurun_out/launches.csv \
  --full gpurun_out/full_r32.ncu-rep:200x100x40/R32 gpurun_out/full_r16.ncu-rep:200x100x40/R16 \
  gpurun_out/full_r8.ncu-rep:200x100x40/R8 gpurun_out/full_r4.ncu-rep:200x100x40/R4 \
  gpurun_out/full_r2.ncu-rep:200x100x40/R2 gpurun_out/full_r1.ncu-rep:200x100x40/R1 > gpurun_out/summary.log 2>&1
mkdir -p gpurun_out/prof_new && cp profiles/r01_launches.* profiles/r01_ncu_full.json profiles/traffic.json gpurun_out/prof_new/
rm -f gpurun_out/full_r16.ncu-rep gpurun_out/full_r8.ncu-rep gpurun_out/full_r4.ncu-rep gpurun_out/full_r2.ncu-rep gpurun_out/full_r1.ncu-rep
du -sh gpurun_out
