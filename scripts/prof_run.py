"""Small driver for ncu captures: one kpm_moments call on a TI lattice.

    python scripts/prof_run.py --lattice 200,100,40 --R 32 --M 8
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lattice", default="200,100,40")
    ap.add_argument("--R", default="32")
    ap.add_argument("--M", type=int, default=8)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--sigma", type=int, default=1)
    ap.add_argument("--variant", default="", help="kernel variant name (KPM_VARIANT by name)")
    ap.add_argument("--order", default="lib", choices=["lib", "ylines", "storage"],
                    help="lib: the library's own order; ylines: workloads.chunk_order_ylines; storage: forced")
    args = ap.parse_args()
    import paper_1410_5242_b200 as kpm

    if args.variant:
        R0 = int(args.R.split(",")[0])
        names = [kpm.variant_name(R0, v) for v in range(32)]
        os.environ["KPM_VARIANT"] = str(names.index(args.variant))
    nx, ny, nz = (int(t) for t in args.lattice.split(","))
    lat = Lattice(nx, ny, nz)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    with kpm.KpmContext(sell_sigma=args.sigma) as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        for R in (int(r) for r in args.R.split(",")):
            if args.order == "storage":
                import numpy as np

                ctx.set_chunk_order(np.arange(ctx.sell_info().n_chunks, dtype=np.int64))
            elif args.order == "ylines":
                import torch

                from workloads.ti_lattice import chunk_order_ylines
                sms = torch.cuda.get_device_properties(0).multi_processor_count
                ctas = {16: 2, 32: 1}.get(R)  # default block-cache feed CTAs per SM (kernels.cu)
                ctx.set_chunk_order(chunk_order_ylines(lat, sms * ctas) if ctas else None)
            for _ in range(args.reps):
                mu, _ = ctx.moments(args.M, R, SEED, want_eta=False)
            t, s, n = ctx.last_timing()
            print(f"R={R} M={args.M} total_ms={t:.3f} sweep_ms={s:.4f} mu0={mu[0]:.0f} kernel={ctx.last_kernel()}",
                  flush=True)


if __name__ == "__main__":
    main()
