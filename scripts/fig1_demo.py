"""Fig. 1-scale demo: DOS of the 1600 x 1600 x 40 topological
insulator (N = 4.1e8; Fig. 1 `topi_dos`) on the GPUs of one box, with
the x-slab distribution and the fused NVLink halo exchange; Jackson-kernel reconstruction.
Run with torchrun (one rank per GPU).  The chunk order is the library's own.  Rank 0 writes
the DOS curve (--out, default gpurun_out/fig1_dos.csv) and prints a JSON summary;
tests/test_gpu_parity.py runs it on a small lattice on one GPU."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, generate_csr_torch, scale_factors  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lattice", default="1600,1600,40")
    ap.add_argument("--M", type=int, default=2000)
    ap.add_argument("--R", type=int, default=32)
    ap.add_argument("--out", default="gpurun_out/fig1_dos.csv")
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    import paper_1410_5242_b200 as kpm

    nx, ny, nz = (int(t) for t in args.lattice.split(","))
    lat = Lattice(nx, ny, nz)
    px = nx // world
    x0, x1 = px * rank, px * (rank + 1)
    t0 = time.time()
    rps, cs, vs = generate_csr(lat, 0, min(21, nx))  # Gershgorin: rows repeat in x (period 20)
    a, b = scale_factors(*gershgorin(rps, cs, vs))
    del rps, cs, vs
    rp, col, val = generate_csr_torch(lat, x0, x1, device=f"cuda:{local}")
    uid = None
    if world > 1:
        box = [kpm.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        uid = box[0]
    ctx = kpm.KpmContext(device=local, nranks=world, rank=rank, nccl_unique_id=uid)
    ctx.set_matrix(rp, col, val, a, b, n_global=lat.n, row_begin=x0 * lat.rows_per_plane, mem=kpm.KPM_MEM_DEVICE)
    del rp, col, val
    torch.cuda.empty_cache()
    t_setup = time.time() - t0
    mu, _ = ctx.moments(args.M, args.R, SEED, want_eta=False)
    total_ms, sweep_ms, _ = ctx.last_timing()
    ctx.close()
    if rank == 0:
        E, rho = kpm.dos(mu, a, b, K=4000)
        os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
        np.savetxt(args.out, np.stack([E, rho], 1), delimiter=",", header="E,rho(E)")
        x = a * (E - b)
        integral = np.pi / len(x) * np.sum(rho / a * np.sqrt(1 - x * x))
        nnz = lat.nnz_expected()
        flops = (args.M // 2) * args.R * (8 * nnz + 34 * lat.n)
        print(json.dumps({"lattice": [nx, ny, nz], "N": lat.n, "N_nz": nnz, "gpus": world, "M": args.M, "R": args.R,
                          "a": a, "b": b, "mu0": mu[0], "integral_rho": integral, "setup_s": t_setup,
                          "moments_s": total_ms / 1e3, "sweep_ms": sweep_ms,
                          "gflops": flops / (total_ms * 1e-3) / 1e9}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
