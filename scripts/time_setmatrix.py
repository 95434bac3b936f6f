"""Time kpm_set_matrix (host CSR) with the device and the host builders; device CSR too."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from workloads.ti_lattice import Lattice, generate_csr, generate_csr_torch, gershgorin, scale_factors  # noqa: E402


def main():
    import paper_1410_5242_b200 as kpm

    lat = Lattice(*(int(t) for t in (sys.argv[1] if len(sys.argv) > 1 else "200,100,40").split(",")))
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    rpd, cold, vald = generate_csr_torch(lat, device="cuda")
    torch.cuda.synchronize()
    for mode in ("0", "1"):
        os.environ["KPM_HOST_BUILD"] = mode
        with kpm.KpmContext() as ctx:
            for rep in range(3):
                t0 = time.perf_counter()
                ctx.set_matrix(rp, col, val, a, b)
                t1 = time.perf_counter()
                print(f"host CSR, KPM_HOST_BUILD={mode}: {1e3 * (t1 - t0):.1f} ms", flush=True)
    os.environ["KPM_HOST_BUILD"] = "0"
    with kpm.KpmContext() as ctx:
        for rep in range(3):
            t0 = time.perf_counter()
            ctx.set_matrix(rpd, cold, vald, a, b, mem=kpm.KPM_MEM_DEVICE)
            t1 = time.perf_counter()
            print(f"device CSR: {1e3 * (t1 - t0):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
