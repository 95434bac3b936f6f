# 4-GPU box: multi-GPU parity (2 and 4 ranks), then Bar weak-scaling bench lines at 2 and 4 GPUs
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29711 \
    bench.py --gpus $n --steps 3 --warmup 3 > gpurun_out/bar_n$n.json 2> gpurun_out/bar_n$n.err; echo "bench n=$n rc=$?"
  cut -c1-300 gpurun_out/bar_n$n.json
done
