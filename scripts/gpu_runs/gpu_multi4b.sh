mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3
for n in 1 2 4; do
if [ $n = 1 ]; then L="python"; else L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n"; fi
timeout 900 $L bench.py --gpus $n --config C4 --steps 3 --warmup 3 --no-e2e --no-r-sweep --no-cpu-baseline > gpurun_out/c4_n$n.json 2> gpurun_out/c4_n$n.err; echo C4 n=$n rc=$?
python -c "import json; d=json.load(open('gpurun_out/c4_n$n.json')); print('C4', $n, d['value'], d['roofline']['sweep_ms'], d['clocks']['sm_mhz'])"
timeout 900 $L bench.py --gpus $n --steps 3 --warmup 3 --no-e2e --no-r-sweep --no-cpu-baseline > gpurun_out/bar_n$n.json 2> gpurun_out/bar_n$n.err; echo bar n=$n rc=$?
python -c "import json; d=json.load(open('gpurun_out/bar_n$n.json')); print('bar', $n, d['value'], d['roofline']['sweep_ms'], d['clocks']['sm_mhz'])"
done
