"""Chunk-order experiment (sustained, power-capped): storage order vs z-column walks, where
CTA b processes the 5 z-blocks of one (x, y) column in consecutive tiles (so a tile's z-runs
come from its own previous / next tile), with board power and SM clock sampled.

    python scripts/exp_order.py <storage|zcol|ylines> <R> <grid>      # on the GPU box (KPM_VARIANT honoured)
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402


def zcol_order(n_chunks, zb, G):
    ncols = n_chunks // zb
    out = []
    for r in range((ncols + G - 1) // G):
        cols = np.arange(r * G, min((r + 1) * G, ncols))
        for z in range(zb):
            out.append(cols * zb + z)
    return np.concatenate(out).astype(np.int64)


def main():
    import paper_1410_5242_b200 as kpm
    mode, R, G = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    lat = Lattice(200, 100, 40)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    with kpm.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        n_chunks = lat.n // 32
        if mode == "zcol":
            ctx.set_chunk_order(zcol_order(n_chunks, 5, G))
        elif mode == "ylines":
            from workloads.ti_lattice import chunk_order_ylines
            ctx.set_chunk_order(chunk_order_ylines(lat, G))
        ctx.moments(8, R, SEED, want_eta=False)
        short = ctx.last_timing()[1]
        t0 = time.time()
        while time.time() - t0 < 5.0:
            mu0, _ = ctx.moments(2000, R, SEED, want_eta=False)
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits",
                                "-i", "0", "-lms", "100"], stdout=subprocess.PIPE, text=True)
        sweeps = []
        for _ in range(4):
            mu, _ = ctx.moments(2000, R, SEED, want_eta=False)
            sweeps.append(ctx.last_timing()[1])
        kern = ctx.last_kernel()
        smi.terminate()
        out = smi.communicate()[0]
    pw, mhz = [], []
    for line in out.splitlines():
        try:
            p, c = (float(x) for x in line.split(","))
            pw.append(p)
            mhz.append(c)
        except ValueError:
            pass
    pw.sort()
    mhz.sort()
    print(json.dumps(dict(order=mode, R=R, grid=G, kernel=kern, short_sweep_ms=short, sweep_ms=sorted(sweeps)[2], power_w=pw[len(pw) // 2],
                          sm_mhz=mhz[len(mhz) // 2], mu2=float(mu[2]))), flush=True)


if __name__ == "__main__":
    main()
