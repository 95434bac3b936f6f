"""P*_LLC probe: the R = 32 sweep on small L2-resident TI lattices (chunk counts that are
multiples of 148 avoid a ragged last wave)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402


def main():
    import paper_1410_5242_b200 as kpm
    for dims in [(20, 24, 40), (37, 8, 40), (37, 12, 40), (37, 16, 40), (74, 4, 40), (37, 4, 40)]:
        lat = Lattice(*dims)
        rp, col, val = generate_csr(lat)
        a, b = scale_factors(*gershgorin(rp, col, val))
        n, nnz = lat.n, int(rp[-1])
        with kpm.KpmContext() as ctx:
            ctx.set_matrix(rp, col, val, a, b)
            res = []
            for M in (200, 2000):
                ctx.moments(M, 32, SEED, want_eta=False)
                ctx.moments(M, 32, SEED, want_eta=False)
                sw = ctx.last_timing()[1]
                res.append(f"M={M}: {sw*1e3:.1f} us {32 * (8 * nnz + 34 * n) / sw / 1e6:.0f} GF/s")
            ws = (32 * 32 * n + 20 * nnz) / 1e6
            print(dims, f"chunks={n // 32} ws={ws:.0f}MB", *res, flush=True)


if __name__ == "__main__":
    main()
