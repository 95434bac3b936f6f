"""A/B of environment knobs of the library (KPM_*) on the default kernel at full size: each
setting in its own process, interleaved in rounds; one JSON line per (round, setting)."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys, subprocess
sys.path.insert(0, %r)
import numpy as np
import paper_1410_5242_b200 as kpm
from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors
nx, ny, nz = %s
R, M = %d, %d
lat = Lattice(nx, ny, nz); rp, col, val = generate_csr(lat); a, b = scale_factors(*gershgorin(rp, col, val))
with kpm.KpmContext() as ctx:
    ctx.set_matrix(rp, col, val, a, b)
    ctx.moments(M, R, SEED, want_eta=False)
    mhz = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
    mu, _ = ctx.moments(M, R, SEED, want_eta=False)
    t, sw, n = ctx.last_timing()
    print(json.dumps(dict(sweep_ms=sw, kernel=ctx.last_kernel(), sm_mhz=mhz, mu1=float(mu[1]))))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lattice", default="200,100,40")
    ap.add_argument("--R", type=int, default=32)
    ap.add_argument("--M", type=int, default=2000)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("settings", nargs="+", help="e.g. KPM_V_EVICT_LAST=0 (use 'default' for none)")
    args = ap.parse_args()
    dims = tuple(int(t) for t in args.lattice.split(","))
    n = 4 * dims[0] * dims[1] * dims[2]
    nnz = 13 * n - 16 * dims[0] * dims[1]
    code = CHILD % (ROOT, dims, args.R, args.M)
    for rnd in range(args.rounds):
        for st in args.settings:
            env = dict(os.environ)
            if st != "default":
                for kv in st.split(","):
                    k, v = kv.split("=")
                    env[k] = v
            out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT)
            line = [l for l in out.stdout.splitlines() if l.startswith("{")]
            d = json.loads(line[-1]) if line else {"error": out.stderr[-500:]}
            if "sweep_ms" in d:
                d["frac"] = (20 * nnz + 48 * args.R * n) / d["sweep_ms"] / 1e6 / 6556.8
            d.update(round=rnd, setting=st)
            print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()
