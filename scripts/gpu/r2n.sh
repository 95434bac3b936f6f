nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_lds_peak scripts/mb_lds_peak.cu && /tmp/mb_lds_peak | tee gpurun_out/r2n_lds_peak.jsonl
nvidia-smi --query-gpu=clocks.sm --format=csv
