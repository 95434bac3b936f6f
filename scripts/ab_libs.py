"""A/B timing of two builds of libkpm.so (e.g. the committed code vs a change) on the default
kernels at full size: each (library, R) in its own process, interleaved in rounds so both see the
same power-capped clock.  One JSON line per (round, library, R): sweep ms, HBM roofline fraction,
SM clock and board power sampled after a warm call, mu[1] (for a same-result check).

    python scripts/ab_libs.py --libs exp/libkpm_old.so,paper_1410_5242_b200/libkpm.so --R 32,16,8
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys, subprocess
sys.path.insert(0, %r)
import paper_1410_5242_b200 as kpm
kpm.LIB_PATH = %r
from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors
nx, ny, nz = %s
R, M = %d, %d
lat = Lattice(nx, ny, nz); rp, col, val = generate_csr(lat); a, b = scale_factors(*gershgorin(rp, col, val))
with kpm.KpmContext() as ctx:
    ctx.set_matrix(rp, col, val, a, b)
    ctx.moments(M, R, SEED, want_eta=False)
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                       capture_output=True, text=True).stdout.strip().split(", ")
    mu, _ = ctx.moments(M, R, SEED, want_eta=False)
    t, sw, n = ctx.last_timing()
    print(json.dumps(dict(sweep_ms=sw, kernel=ctx.last_kernel(), sm_mhz=q[0], power_w=q[-1], mu1=float(mu[1]))))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True, help="comma list of libkpm.so paths")
    ap.add_argument("--R", default="32,16,8")
    ap.add_argument("--M", type=int, default=2000)
    ap.add_argument("--lattice", default="200,100,40")
    ap.add_argument("--rounds", type=int, default=3)
    args = ap.parse_args()
    nx, ny, nz = (int(t) for t in args.lattice.split(","))
    n = 4 * nx * ny * nz
    nnz = 13 * n - 16 * nx * ny
    hbm = 6556.8
    peaks = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks):
        hbm = json.load(open(peaks)).get("hbm_gbs", hbm)
    for rnd in range(args.rounds):
        for R in (int(r) for r in args.R.split(",")):
            for lib in args.libs.split(","):
                code = CHILD % (ROOT, os.path.abspath(lib), (nx, ny, nz), R, args.M)
                res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900)
                try:
                    row = json.loads(res.stdout.strip().splitlines()[-1])
                except Exception:
                    print(json.dumps(dict(round=rnd, R=R, lib=lib, error=res.stderr[-400:])), flush=True)
                    continue
                alg = 20 * nnz + 48 * R * n
                row.update(round=rnd, R=R, lib=lib, frac=alg / (row["sweep_ms"] * 1e-3) / 1e9 / hbm)
                print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
