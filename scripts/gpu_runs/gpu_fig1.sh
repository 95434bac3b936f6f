mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 scripts/fig1_demo.py > gpurun_out/fig1.json 2> gpurun_out/fig1.err; echo rc=$?
cat gpurun_out/fig1.json; tail -3 gpurun_out/fig1.err
