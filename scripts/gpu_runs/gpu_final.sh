# refresh: plain bench line (default flags), then the profiles (launch list + ncu --set full per R)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
bash scripts/profile_round.sh
