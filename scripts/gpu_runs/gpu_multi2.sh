mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -15
for mode in fused nccl; do
KPM_HALO=$mode timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_n2_$mode.json 2> gpurun_out/bench_n2_$mode.err; echo mode=$mode rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_n2_$mode.json')); print('$mode', d['value'], d['roofline']['sweep_ms'], d['clocks'])"
done
