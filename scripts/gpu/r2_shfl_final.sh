# Shuffle/LDS concurrency microbenchmark, then the full validation (GPU tests, smoke, bench, reference arm)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_shfl scripts/mb_shfl.cu && timeout 120 /tmp/mb_shfl > gpurun_out/mb_shfl.jsonl 2>&1; echo "mb rc=$?"
bash scripts/gpu/r2_final.sh
