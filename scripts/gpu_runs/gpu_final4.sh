# 4-GPU box, final state: full GPU test suite (incl. 2- and 4-rank parity and the C4 Bloch pins),
# smoke, then Bar weak-scaling bench lines at 1, 2 and 4 GPUs
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/f4_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/f4_pytest.log | head -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/f4_n1.json 2> gpurun_out/f4_n1.err; echo "bench n=1 rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2973$n \
    bench.py --gpus $n --steps 3 --warmup 3 > gpurun_out/f4_n$n.json 2> gpurun_out/f4_n$n.err; echo "bench n=$n rc=$?"
done
for n in 1 2 4; do python -c "
import json; d=json.load(open('gpurun_out/f4_n$n.json'))
print($n, round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['config']['kernel_variant'], d['config']['chunk_order'], round(d['e2e']['value']) if d.get('e2e') else None)"; done
