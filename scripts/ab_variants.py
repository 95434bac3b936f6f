"""A/B timing of sweep-kernel variants at full size (C3 by default), interleaved in rounds so
that all see the same power-capped clock; by default each runs in the chunk order the library
picks for it.  One JSON line per (round, R, variant): sweep ms, HBM roofline fraction, deviation
of mu from the round's first variant, SM clock and board power sampled after a warm call."""
import argparse
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from workloads.ti_lattice import SEED, Lattice, chunk_order_ylines, gershgorin, generate_csr, scale_factors  # noqa: E402


def clock():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=10).stdout.strip().split(", ")
        return float(out[0]), float(out[1])
    except Exception:
        return None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lattice", default="200,100,40")
    ap.add_argument("--R", default="32,16,8")
    ap.add_argument("--M", type=int, default=2000)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--names", default="", help="comma list of variant names (default: all of the width)")
    ap.add_argument("--order", default="lib", choices=["ylines", "none", "lib", "ystrips", "ystrips3", "ystrips4"],
                    help="lib: the library's own chunk order; ylines: workloads.chunk_order_ylines; none: storage")
    args = ap.parse_args()
    import torch

    import paper_1410_5242_b200 as kpm

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    nx, ny, nz = (int(t) for t in args.lattice.split(","))
    lat = Lattice(nx, ny, nz)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    n, nnz = lat.n, int(rp[-1])
    hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6556.8
    for rnd in range(args.rounds):
        for R in (int(r) for r in args.R.split(",")):
            names = [kpm.variant_name(R, v) for v in range(32) if kpm.variant_name(R, v)]
            want = args.names.split(",") if args.names else names
            ref = None
            for name in want:
                if name not in names:
                    continue
                v = names.index(name)
                os.environ["KPM_VARIANT"] = str(v)
                with kpm.KpmContext() as ctx:
                    ctx.set_matrix(rp, col, val, a, b)
                    if args.order == "ylines" and ".bc." in name:
                        per_sm = 1 if R == 32 else (2 if R == 16 else 3)
                        ctx.set_chunk_order(chunk_order_ylines(lat, sms * per_sm))
                    elif args.order.startswith("ystrips") and ".bc." in name:
                        from workloads.ti_lattice import chunk_order_ystrips

                        per_sm = 1 if R == 32 else (2 if R == 16 else 3)
                        width = int(args.order[7:] or 2)
                        ctx.set_chunk_order(chunk_order_ystrips(lat, sms * per_sm, width=width))
                    elif args.order == "none":
                        ctx.set_chunk_order(np.arange(ctx.sell_info().n_chunks, dtype=np.int64))
                    ctx.moments(args.M, R, SEED, want_eta=False)
                    mhz, watt = clock()
                    mu, _ = ctx.moments(args.M, R, SEED, want_eta=False)
                    ran = ctx.last_kernel()
                    t, sw, ns = ctx.last_timing()
                if ref is None:
                    ref = mu
                bytes_ = 20 * nnz + 48 * R * n
                row = dict(round=rnd, R=R, variant=name, order=args.order, ran=ran, sweep_ms=sw, frac=bytes_ / sw / 1e6 / hbm,
                           gflops=R * (8 * nnz + 34 * n) / sw / 1e6, dmu=float(np.max(np.abs(mu - ref)) / ref[0]),
                           sm_mhz=mhz, power_w=watt, lattice=[nx, ny, nz], M=args.M, time=time.time())
                print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
