nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_pipes scripts/mb_pipes.cu && /tmp/mb_pipes | tee gpurun_out/r2l_pipes.jsonl
