"""Phase timing of the bench's e2e step (kpm_set_matrix from host CSR + kpm_moments)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from workloads.ti_lattice import SEED, Lattice, generate_csr, gershgorin, scale_factors  # noqa: E402


def main():
    import paper_1410_5242_b200 as kpm

    lat = Lattice(200, 100, 40)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    with kpm.KpmContext(cuda_stream=stream.cuda_stream) as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        ctx.moments(2000, 32, SEED)
        for rep in range(3):
            t0 = time.perf_counter()
            ctx.set_matrix(rp, col, val, a, b)
            t1 = time.perf_counter()
            ctx.moments(2000, 32, SEED, want_eta=True)
            t2 = time.perf_counter()
            print(f"set_matrix {1e3*(t1-t0):.1f} ms  moments {1e3*(t2-t1):.1f} ms  (device total {ctx.last_timing()[0]:.1f})", flush=True)
        pinned = [torch.from_numpy(x).pin_memory() for x in (rp, col, val)]
        prp, pcol, pval = (t.numpy() for t in pinned)
        for rep in range(3):
            t0 = time.perf_counter()
            ctx.set_matrix(prp, pcol, pval, a, b)
            t1 = time.perf_counter()
            print(f"pinned set_matrix {1e3*(t1-t0):.1f} ms", flush=True)
        for rep in range(2):
            t1 = time.perf_counter()
            ctx.moments(2000, 32, SEED, want_eta=True)
            t2 = time.perf_counter()
            print(f"moments only {1e3*(t2-t1):.1f} ms (device total {ctx.last_timing()[0]:.1f})", flush=True)


if __name__ == "__main__":
    main()
