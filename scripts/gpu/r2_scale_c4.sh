# C4 strong scaling re-check on a 4-GPU box after the leftover-segment chunk order
mkdir -p gpurun_out/scale4b
run() { local n=$1; shift; local tag=$1; shift
  if [ "$n" = 1 ]; then timeout 1200 python bench.py --gpus 1 "$@" > gpurun_out/scale4b/${tag}_n1.json 2> gpurun_out/scale4b/${tag}_n1.err
  else timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800 + n)) bench.py --gpus $n "$@" > gpurun_out/scale4b/${tag}_n$n.json 2> gpurun_out/scale4b/${tag}_n$n.err; fi
  echo "$tag n=$n rc=$?"; }
for n in 1 2 4; do run $n c4 --config C4 --steps 3 --warmup 3 --no-r-sweep --no-cpu-baseline --no-e2e; done
run 4 bar --steps 5 --warmup 3 --no-r-sweep --no-e2e
grep -h "NCCL INFO" gpurun_out/scale4b/bar_n4.err | head -12
