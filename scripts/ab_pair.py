"""A/B timing of sweep-kernel variants at full size (C3 by default), interleaved in rounds so
that both see the same power-capped clock; y-line chunk order sized to each variant's grid.
One JSON line per (round, R, variant): sweep ms, HBM roofline fraction, deviation of mu."""
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
    ap.add_argument("--order", default="ylines", choices=["ylines", "none", "lib"])
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
    ctas = {"tiled.bc.lpr8.u4": 1, "tiled.bc.lpr4.u4.wr": None}
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
                        per_sm = 1 if name.startswith("pair") or R == 32 else (2 if R == 16 else 3)
                        ctx.set_chunk_order(chunk_order_ylines(lat, sms * per_sm))
                    ctx.moments(args.M, R, SEED, want_eta=False)
                    mhz, watt = clock()
                    mu, _ = ctx.moments(args.M, R, SEED, want_eta=False)
                    ran = ctx.last_kernel()
                    t, sw, ns = ctx.last_timing()
                if ref is None:
                    ref = mu
                bytes_ = 20 * nnz + 48 * R * n
                row = dict(round=rnd, R=R, variant=name, ran=ran, sweep_ms=sw, frac=bytes_ / sw / 1e6 / hbm,
                           gflops=R * (8 * nnz + 34 * n) / sw / 1e6, dmu=float(np.max(np.abs(mu - ref)) / ref[0]),
                           sm_mhz=mhz, power_w=watt, lattice=[nx, ny, nz], M=args.M, time=time.time())
                print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
