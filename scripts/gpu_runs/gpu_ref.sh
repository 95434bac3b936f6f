mkdir -p gpurun_out
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_n1.json 2> gpurun_out/ref_n1.err; echo ref1 rc=$?; cat gpurun_out/ref_n1.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/ref_n2.json 2> gpurun_out/ref_n2.err; echo ref2 rc=$?; cat gpurun_out/ref_n2.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29912 bench.py --gpus 2 > gpurun_out/bench_n2d.json 2> gpurun_out/bench_n2d.err; echo bench2 rc=$?; wc -l gpurun_out/bench_n2d.json; cut -c1-400 gpurun_out/bench_n2d.json
