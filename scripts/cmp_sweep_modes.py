"""Sweep time in kpm_moments (V/W swap every sweep) vs kpm_sweep_kernel('aug') (fixed V)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402


def main():
    import paper_1410_5242_b200 as kpm
    lat = Lattice(200, 100, 40)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    with kpm.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        for R in (4, 8, 16, 32):
            for rep in range(2):
                ctx.moments(200, R, SEED, want_eta=False)
                sw = ctx.last_timing()[1]
                ms, _ = ctx.sweep_kernel("aug", R, SEED, n_sweeps=99)
                print(f"R={R} rep={rep} moments sweep {sw:.4f} ms   sweep_kernel aug {ms:.4f} ms  {ctx.last_kernel()}", flush=True)


if __name__ == "__main__":
    main()
