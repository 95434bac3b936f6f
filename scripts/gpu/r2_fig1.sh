nvidia-smi --query-gpu=index,clocks.sm,power.draw --format=csv
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 scripts/fig1_demo.py --out gpurun_out/r02_fig1_dos.csv > gpurun_out/r02_fig1.json 2> gpurun_out/r02_fig1.err; echo "rc=$?"
tail -c 700 gpurun_out/r02_fig1.json
