"""Multi-GPU parity, launched by tests/test_gpu_multi.py under torchrun (one rank per GPU).

Each rank owns an x-slab of the TI lattice (the row distribution of PAPER.md P:849-854) and
runs kpm_moments with the NCCL halo exchange; rank 0 checks the moments against the oracle
on the global matrix (1e-10 gate) and against a single-rank run (P-invariance)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import sell_ref  # noqa: E402
from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402

TOL = 1e-10


def random_hermitian(n, per_row, seed):
    """Seeded irregular sparse Hermitian CSR (row lengths vary, columns anywhere)."""
    rng = np.random.default_rng(seed)
    i = np.repeat(np.arange(n), rng.integers(1, per_row + 1, size=n))
    j = rng.integers(0, n, size=i.size)
    v = rng.normal(size=i.size) + 1j * rng.normal(size=i.size)
    rows = np.concatenate([i, j, np.arange(n)])
    cols = np.concatenate([j, i, np.arange(n)])
    vals = np.concatenate([v, np.conj(v), rng.normal(size=n) + 0j])
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    return np.cumsum(rp), cols.astype(np.int64), vals


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    import paper_1410_5242_b200 as kpm

    uid = [kpm.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    results, mu_by_case = {}, {}
    cases = [((8, 8, 8), 64, 4, SEED), ((12, 5, 8), 80, 32, 7), ((10, 3, 5), 40, 5, 11), ((6, 4, 16), 200, 16, 3),
             ((12, 6, 16), 60, 32, "device"), ((max(3, world), 5, 8), 40, 8, 17), ("random", 60, 8, 19)]
    ctx = kpm.KpmContext(device=local, nranks=world, rank=rank, nccl_unique_id=uid[0])
    for (dims, M, R, seed), mode in [(c, m) for m in ("fused", "nccl") for c in cases]:
        os.environ["KPM_HALO"] = mode  # read by kpm_set_matrix
        if dims == "random":
            # irregular Hermitian matrix, uneven row split: every rank exchanges with every
            # other, halo runs are scattered (not x-planes)
            n_g = 2900
            rp_g, col_g, val_g = random_hermitian(n_g, 9, 23)
            bounds = [0] + [int(n_g * f) for f in np.cumsum(np.arange(1, world + 1) / np.arange(1, world + 1).sum())]
            bounds[-1] = n_g
            r0, r1 = bounds[rank], bounds[rank + 1]
        else:
            lat = Lattice(*dims)
            n_g = lat.n
            planes = [lat.nx * q // world for q in range(world + 1)]
            rp_g, col_g, val_g = generate_csr(lat)
            r0, r1 = planes[rank] * lat.rows_per_plane, planes[rank + 1] * lat.rows_per_plane
        a, b = scale_factors(*gershgorin(rp_g, col_g, val_g))
        if seed == "device":  # CSR generated and converted on the GPU (KPM_MEM_DEVICE)
            from workloads.ti_lattice import generate_csr_torch

            seed = 13
            rp, col, val = generate_csr_torch(lat, planes[rank], planes[rank + 1], device=f"cuda:{local}")
            ctx.set_matrix(rp, col, val, a, b, n_global=n_g, row_begin=r0, mem=kpm.KPM_MEM_DEVICE)
        else:
            rp = rp_g[r0:r1 + 1] - rp_g[r0]
            col, val = col_g[rp_g[r0]:rp_g[r1]], val_g[rp_g[r0]:rp_g[r1]]
            ctx.set_matrix(rp, col, val, a, b, n_global=n_g, row_begin=r0)
        # the rank's SELL copy and halo map, bit-exact against the numpy reference builder
        bounds_all = np.array(bounds if dims == "random" else [q * lat.rows_per_plane for q in planes], dtype=np.int64)
        ref = sell_ref.build_sell(rp_g[r0:r1 + 1] - rp_g[r0], col_g[rp_g[r0]:rp_g[r1]], val_g[rp_g[r0]:rp_g[r1]],
                                  row_begin=r0, row_end=r1, row_begins=bounds_all)
        ex = ctx.export_sell()
        sell_ok = all(np.array_equal(ex[k], ref[k]) for k in ("cptr", "col", "val", "perm", "halo"))
        sell_all = [None] * world
        dist.all_gather_object(sell_all, bool(sell_ok))
        mu, eta = ctx.moments(M, R, seed)
        if mode == "fused":
            mu_by_case[dims] = mu
        # explicit v0 path (halo of nu_0 exchanged instead of generated)
        rng = np.random.default_rng(5)
        v0_g = rng.normal(size=(n_g, 2)) + 1j * rng.normal(size=(n_g, 2))
        mu_v, eta_v = ctx.moments_v0(M, v0_g[r0:r1])
        gathered = [None] * world
        dist.all_gather_object(gathered, (mu.tolist(), mu_v.tolist()))
        if rank == 0:
            import oracle

            eta_o = oracle.kpm_eta(rp_g, col_g, val_g, a, b, M, R, seed)
            mu_o, _ = oracle.eta_to_mu(eta_o)
            eta_vo = oracle.kpm_eta_v0(rp_g, col_g, val_g, a, b, M, v0_g)
            mu_vo, _ = oracle.eta_to_mu(eta_vo)
            col_err = float(np.max(np.abs(eta - eta_o) / eta_o[:, :1].real))
            mu_err = float(np.max(np.abs(mu - mu_o)) / mu_o[0])
            v_err = float(np.max(np.abs(eta_v - eta_vo) / eta_vo[:, :1].real))
            same = all(np.array_equal(np.array(g[0]), mu) for g in gathered)
            results[f"{dims}/{mode}"] = dict(col_err=col_err, mu_err=mu_err, v0_err=v_err, ranks_identical=bool(same),
                                             sell_halo_exact=all(sell_all),
                                             ok=bool(col_err <= TOL and mu_err <= TOL and v_err <= TOL and same
                                                     and all(sell_all)))
    ctx.close()
    if rank == 0:
        # P-invariance against a single-rank context on the same device
        lat = Lattice(12, 5, 8)
        rp_g, col_g, val_g = generate_csr(lat)
        a, b = scale_factors(*gershgorin(rp_g, col_g, val_g))
        with kpm.KpmContext(device=local) as c1:
            c1.set_matrix(rp_g, col_g, val_g, a, b)
            mu1, _ = c1.moments(80, 32, 7)
        err = float(np.max(np.abs(mu_by_case[(12, 5, 8)] - mu1)) / mu1[0])
        results["p_invariance"] = dict(err=err, ok=bool(err <= TOL))
        out = dict(world=world, cases=results)
        print("MGPU_RESULT " + json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
