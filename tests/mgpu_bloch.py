"""Full-size multi-GPU pin, launched by tests/test_gpu_multi.py under torchrun: the C4
lattice (400x400x40, N = 25.6M) at V = 0, x-slab row partition over the ranks, R = 32
Z4 vectors, M moments; rank 0 compares mu with the exact trace from the partial-Bloch
spectrum (tests/bloch_ref.py; SURVEY §8(c) "open-z, large N"): |mu_n - tr T_n| <= 6 sigma_n
with sigma_n^2 <= sum_k T_n(x_k)^2 / R, and mu_0 = N exactly."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from workloads.ti_lattice import SEED, ZERO_POTENTIAL, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    import paper_1410_5242_b200 as kpm

    dims = tuple(int(t) for t in os.environ.get("MGPU_BLOCH_DIMS", "400,400,40").split(","))
    M, R = 200, 32
    lat = Lattice(*dims, potential=ZERO_POTENTIAL)
    planes = [lat.nx * q // world for q in range(world + 1)]
    rp, col, val = generate_csr(lat, planes[rank], planes[rank + 1])
    r0 = planes[rank] * lat.rows_per_plane
    lo, hi = gershgorin(rp, col, val, row_begin=r0)
    t = torch.tensor([-lo, hi], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    a, b = scale_factors(-float(t[0]), float(t[1]))
    uid = [kpm.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    with kpm.KpmContext(device=local, nranks=world, rank=rank, nccl_unique_id=uid[0]) as ctx:
        ctx.set_matrix(rp, col, val, a, b, n_global=lat.n, row_begin=r0)
        mu, _ = ctx.moments(M, R, SEED, want_eta=False)
    if rank == 0:
        from bloch_ref import cheb_moments, slab_energies

        x = a * (slab_energies(lat, rp, col, val) - b)  # rank 0's rows start with site column (0, 0)
        tr, sq = cheb_moments(x, M)
        z = np.abs(mu - tr) / np.sqrt(sq / R)
        out = dict(world=world, dims=dims, n=lat.n, mu0_exact=bool(mu[0] == lat.n), max_z=float(np.max(z[1:])),
                   rms_z=float(np.sqrt(np.mean(z[1:] ** 2))), xmax=float(np.max(np.abs(x))))
        out["ok"] = bool(out["mu0_exact"] and out["max_z"] < 6.0 and out["rms_z"] < 1.5 and out["xmax"] < 1)
        print("MGPU_BLOCH " + json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
