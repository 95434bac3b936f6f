"""Time every aug_spmmv variant per block width on a TI lattice (tuning; KPM_VARIANT)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lattice", default="200,100,40")
    ap.add_argument("--R", default="1,2,4,8,16,32")
    ap.add_argument("--M", type=int, default=40)
    ap.add_argument("--grid-per-sm", default="0")
    ap.add_argument("--variants", default="", help="comma list of variant indices (default: all)")
    ap.add_argument("--warm-seconds", type=float, default=0.0, help="run this long before timing (power-cap steady state)")
    args = ap.parse_args()
    import paper_1410_5242_b200 as kpm

    nx, ny, nz = (int(t) for t in args.lattice.split(","))
    lat = Lattice(nx, ny, nz)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    n, nnz = lat.n, int(rp[-1])
    res = []
    for R in (int(r) for r in args.R.split(",")):
        ref = None
        names = set()
        vlist = [int(x) for x in args.variants.split(",")] if args.variants else range(16)
        for v in vlist:
            for g in args.grid_per_sm.split(","):
                os.environ["KPM_VARIANT"] = str(v)
                os.environ["KPM_GRID_PER_SM"] = g
                with kpm.KpmContext() as ctx:
                    ctx.set_matrix(rp, col, val, a, b)
                    import time as _t
                    t0 = _t.time()
                    ctx.moments(args.M, R, SEED, want_eta=False)
                    while _t.time() - t0 < args.warm_seconds:
                        ctx.moments(args.M, R, SEED, want_eta=False)
                    mu, _ = ctx.moments(args.M, R, SEED, want_eta=False)
                    name = ctx.last_kernel()
                    t, sw, ns = ctx.last_timing()
                if not args.variants and v > 0 and name in names and g == args.grid_per_sm.split(",")[0]:
                    break
                names.add(name)
                if ref is None:
                    ref = mu
                err = float(np.max(np.abs(mu - ref)) / ref[0])
                bytes_ = 20 * nnz + 48 * R * n
                row = dict(R=R, v=v, grid_per_sm=g, kernel=name, sweep_ms=sw, gbs=bytes_ / sw / 1e6,
                           frac=bytes_ / sw / 1e6 / 6450, gflops=R * (8 * nnz + 34 * n) / sw / 1e6, dmu=err)
                res.append(row)
                print(json.dumps(row), flush=True)
            else:
                continue
            break


if __name__ == "__main__":
    main()
