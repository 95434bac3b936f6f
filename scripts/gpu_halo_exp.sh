# per-sweep cost of the halo exchange at 2 GPUs (Bar weak, C3 slab per GPU), M=400.
# The "fused_no_peer_stores" line needs a measurement-only build in which kpm_abi.cu's
# fused sweep sets sa.n_peer = 0 when env KPM_EXP_NO_PEER=1 (results wrong; timing only);
# with the product library it repeats the "fused" case.
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 2 --steps 3 --warmup 3 --M 400 --no-e2e --no-r-sweep --no-cpu-baseline"
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['roofline']['sweep_ms'],4), round(d['value']))"; }
$R --master-port 29701 $B 2>/dev/null | show fused
KPM_EXP_NO_PEER=1 $R --master-port 29702 $B 2>/dev/null | show fused_no_peer_stores
KPM_HALO=nccl $R --master-port 29703 $B 2>/dev/null | show nccl
CUDA_VISIBLE_DEVICES=0 python bench.py --steps 3 --warmup 3 --M 400 --no-e2e --no-r-sweep --no-cpu-baseline 2>/dev/null | show single
