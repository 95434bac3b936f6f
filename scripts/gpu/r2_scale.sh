# Multi-GPU evidence with the final defaults on an N-GPU box (N = $1): multi-rank tests, then
# Bar weak / C4 strong / C5 weak bench lines at 1..N GPUs on the same box (NCCL INIT on stderr).
NG=${1:-2}
mkdir -p gpurun_out/scale$NG
nvidia-smi --query-gpu=index,name,clocks.sm,power.draw,power.limit --format=csv
nvidia-smi topo -m > gpurun_out/scale$NG/topo.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_virtual.py -x -q > gpurun_out/scale$NG/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/scale$NG/pytest.log
run() {  # run N tag args...
  local n=$1; shift; local tag=$1; shift
  if [ "$n" = 1 ]; then
    timeout 1800 python bench.py --gpus 1 "$@" > gpurun_out/scale$NG/${tag}_n1.json 2> gpurun_out/scale$NG/${tag}_n1.err
  else
    timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + n)) \
      bench.py --gpus $n "$@" > gpurun_out/scale$NG/${tag}_n$n.json 2> gpurun_out/scale$NG/${tag}_n$n.err
  fi
  echo "$tag n=$n rc=$? $(tail -c 300 gpurun_out/scale$NG/${tag}_n$n.json)"
}
for n in 1 2 4; do [ $n -le $NG ] && run $n bar --steps 5 --warmup 3 --no-r-sweep; done
for n in 1 2 4; do [ $n -le $NG ] && run $n c4 --config C4 --steps 3 --warmup 3 --no-r-sweep --no-cpu-baseline --no-e2e; done
run 1 c5 --config C5 --steps 2 --warmup 3 --no-r-sweep --no-cpu-baseline --no-e2e
run $NG c5 --config C5 --steps 2 --warmup 3 --no-r-sweep --no-cpu-baseline --no-e2e
grep -h "NCCL INFO.*\(nranks\|comm \|Init COMPLETE\|NVLS\|P2P\)" gpurun_out/scale$NG/*_n$NG.err | head -20
