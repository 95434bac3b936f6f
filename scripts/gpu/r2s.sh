export KPM_TRACE=1
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29721 tests/mgpu_failure.py > gpurun_out/r2s_out.log 2> gpurun_out/r2s_err.log; echo "rc=$?"
grep -h "MGPU_FAILURE" gpurun_out/r2s_out.log; grep -h "kpm r0" gpurun_out/r2s_err.log | tail -15
