"""Sustained (power-capped) sweep time, SM clock and board power of the R = 32 sweep with
parts of the on-chip work removed (timing only, wrong results): exp/libkpm_eN.so from
scripts/exp_bottleneck.py --build (N = 0 product, 1 no non-own V copies, 2 no shared-memory
V gathers, 3 both).  Shows how much of a traffic cut turns into clock under the 1 kW cap.

    python scripts/exp_power.py 1        # on the GPU box
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402


def main():
    import paper_1410_5242_b200 as kpm
    e = sys.argv[1]
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    kpm.LIB_PATH = os.path.join(ROOT, "exp", f"libkpm_e{e}.so")
    lat = Lattice(200, 100, 40)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    with kpm.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        t0 = time.time()
        while time.time() - t0 < 5.0:  # reach the power-capped steady state
            ctx.moments(2000, R, SEED, want_eta=False)
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits",
                                "-i", "0", "-lms", "100"], stdout=subprocess.PIPE, text=True)
        sweeps = []
        for _ in range(4):
            mu, _ = ctx.moments(2000, R, SEED, want_eta=False, allow_warning=True)
            sweeps.append(ctx.last_timing()[1])
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
    print(json.dumps(dict(exp=int(e), R=R, sweep_ms=sorted(sweeps)[len(sweeps) // 2],
                          power_w=pw[len(pw) // 2] if pw else None, sm_mhz=mhz[len(mhz) // 2] if mhz else None,
                          samples=len(pw), mu2=float(mu[2]), mu_last=float(mu[-1]))), flush=True)


if __name__ == "__main__":
    main()
