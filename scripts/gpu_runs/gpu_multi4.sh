mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; echo n=$n rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_n$n.json')); print($n, d['value'], d['roofline']['sweep_ms'], d['clocks'])"
done
