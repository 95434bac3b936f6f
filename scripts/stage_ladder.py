"""The paper's optimisation-stage ladder on one B200 (Fig. 11 / Table III analogue):
naive BLAS-1 chain (Fig. 3), aug_spmv column by column (Fig. 4, = throughput mode),
aug_spmmv blocked (Fig. 5); same lattice, same R random vectors, Gflop/s in the paper's
algorithmic currency.  Prints one JSON line."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lattice", default="200,100,40")
    ap.add_argument("--M", type=int, default=200)
    ap.add_argument("--R", type=int, default=32)
    args = ap.parse_args()
    import paper_1410_5242_b200 as kpm

    lat = Lattice(*(int(t) for t in args.lattice.split(",")))
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    n, nnz = lat.n, int(rp[-1])
    flops = (args.M // 2) * args.R * (8 * nnz + 34 * n)
    out = {"lattice": list(lat.__dict__.values())[:3], "M": args.M, "R": args.R, "stages": {}}
    with kpm.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        for st in ("naive", "aug_spmv", "aug_spmmv"):
            ctx.moments_stage(st, args.M, args.R, SEED, want_eta=False)  # warm-up
            mu, _ = ctx.moments_stage(st, args.M, args.R, SEED, want_eta=False)
            t_ms = ctx.last_timing()[0]
            out["stages"][st] = {"ms": t_ms, "gflops": flops / (t_ms * 1e-3) / 1e9, "kernel": ctx.last_kernel(),
                                 "mu1": mu[1]}
    base = out["stages"]["naive"]["ms"]
    for st in out["stages"].values():
        st["speedup_vs_naive"] = base / st["ms"]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
