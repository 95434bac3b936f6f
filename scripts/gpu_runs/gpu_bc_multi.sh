# block cache on several ranks: multi-GPU parity (2 ranks) and the Bar weak-scaling bench at 2 GPUs
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -k "parity" > gpurun_out/bcm_pytest.log 2>&1; echo "mgpu pytest rc=$?"; tail -3 gpurun_out/bcm_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29721 \
  bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bcm_n2.json 2> gpurun_out/bcm_n2.err; echo "bench n=2 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bcm_n2.json'))
print(d['value'], d['roofline']['frac'], d['clocks'], d['config']['kernel_variant'], d['config']['chunk_order'])"
