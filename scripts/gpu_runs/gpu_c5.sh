mkdir -p gpurun_out
( timeout 1500 python bench.py --config C5 --steps 1 --warmup 1 --no-r-sweep > gpurun_out/c5_n1.json 2> gpurun_out/c5_n1.err; echo C5 rc=$? ) 
tail -5 gpurun_out/c5_n1.err
cat gpurun_out/c5_n1.json
