"""Virtual-rank parity cases (KPM_VIRTUAL_RANKS), run by tests/test_gpu_virtual.py in a
subprocess whose environment sets CUDA_DEVICE_MAX_CONNECTIONS (one hardware queue per stream)
and whose timeout bounds a hang.  usage: python tests/vranks_parity.py ti P R | uneven P | mismatch
Prints one line "VRANKS_RESULT {json}"."""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from oracle import sell_ref  # noqa: E402
from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402

TOL = 1e-10


def run_ranks(pkg, P, fn, timeout=600):
    """fn(ctx, rank) on P virtual ranks in P threads; returns the per-rank results."""
    group = pkg.VirtualGroup(P)
    out, err = [None] * P, [None] * P

    def worker(r):
        try:
            with pkg.KpmContext(device=0, nranks=P, rank=r, vgroup=group) as ctx:
                out[r] = fn(ctx, r)
        except BaseException as e:  # noqa: BLE001 -- reported below
            err[r] = e

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(P)]
    for t in th:
        t.start()
    deadline = time.time() + timeout
    for t in th:
        t.join(max(0.0, deadline - time.time()))
    assert not any(t.is_alive() for t in th), "virtual ranks hung"
    group.close()
    for e in err:
        if e is not None:
            raise e
    return out


def ti_problem(dims):
    lat = Lattice(*dims)
    rp, col, val = generate_csr(lat)
    return lat, rp, col, val


def mixed_problem(P):
    """TI lattice plus seeded random long-range Hermitian couplings among rank 1's rows: rank 1's
    chunks read scattered rows (its tile / block-cache plans do not fit), the others stay
    stencil-like, so the ranks must agree on a kernel variant every rank can run."""
    lat, rp, col, val = ti_problem((4 * P, 5, 16))
    n = lat.n
    r0, r1 = n // P, 2 * n // P
    rng = np.random.default_rng(41)
    i = rng.integers(r0, r1, 600)
    j = rng.integers(r0, r1, 600)
    z = 0.05 * (rng.normal(size=600) + 1j * rng.normal(size=600))
    import scipy.sparse as sp

    h = sp.csr_matrix((val, col, rp), shape=(n, n)) + sp.coo_matrix((z, (i, j)), shape=(n, n)).tocsr()
    h = (h + sp.coo_matrix((np.conj(z), (j, i)), shape=(n, n)).tocsr()).tocsr()
    h.sort_indices()
    return n, h.indptr.astype(np.int64), h.indices.astype(np.int64), h.data.astype(np.complex128)


def check(mu_g, eta_g, eta_o):
    mu_o, _ = oracle.eta_to_mu(eta_o)
    assert np.max(np.abs(eta_g - eta_o) / eta_o[:, :1].real) <= TOL
    assert np.max(np.abs(mu_g - mu_o)) / mu_o[0] <= TOL


def run_case(pkg, P, n, rp, col, val, bounds, M, R, seed, want_v0=False):
    a, b = scale_factors(*gershgorin(rp, col, val))
    rng = np.random.default_rng(5)
    v0 = rng.normal(size=(n, 2)) + 1j * rng.normal(size=(n, 2))

    def fn(ctx, r):
        trace = os.environ.get("VRANKS_TRACE")
        r0, r1 = bounds[r], bounds[r + 1]
        lrp = rp[r0:r1 + 1] - rp[r0]
        lcol, lval = col[rp[r0]:rp[r1]], val[rp[r0]:rp[r1]]
        ctx.set_matrix(lrp, lcol, lval, a, b, n_global=n, row_begin=r0)
        if trace:
            print(f"rank {r}: set_matrix done", flush=True)
        mu, eta = ctx.moments(M, R, seed)
        if trace:
            print(f"rank {r}: moments done ({ctx.last_kernel()})", flush=True)
        res = dict(mu=mu, eta=eta, kernel=ctx.last_kernel(), sell=ctx.export_sell(), halo=ctx.export_halo(), lrp=lrp,
                   lcol=lcol, lval=lval)
        if want_v0:
            res["v0"] = ctx.moments_v0(M, v0[r0:r1])
        return res

    out = run_ranks(pkg, P, fn)
    eta_o = oracle.kpm_eta(rp, col, val, a, b, M, R, seed)
    for r, o in enumerate(out):
        check(o["mu"], o["eta"], eta_o)
        assert np.array_equal(o["mu"], out[0]["mu"])  # identical on every rank (one reduction)
        assert o["kernel"] == out[0]["kernel"]          # every rank ran the same variant
        r0, r1 = bounds[r], bounds[r + 1]
        ref = sell_ref.build_sell(o["lrp"], o["lcol"], o["lval"], row_begin=r0, row_end=r1,
                                  row_begins=np.asarray(bounds))
        for k in ("cptr", "col", "val", "perm", "halo"):
            assert np.array_equal(o["sell"][k], ref[k]), (r, k)
        recv = pkg.plan_recv(np.asarray(bounds), r, o["lrp"], o["lcol"])
        assert np.array_equal(o["halo"][0], recv)  # kpm_export_halo == the host planner
    if want_v0:
        eta_vo = oracle.kpm_eta_v0(rp, col, val, a, b, M, v0)
        for o in out:
            mu_v, eta_v = o["v0"]
            assert np.max(np.abs(eta_v - eta_vo) / eta_vo[:, :1].real) <= TOL
    return out


def case_ti(pkg, P, R):
    """x-slabs of a TI lattice (2 planes per rank at P = 8): the default kernels (block-cache feed
    at R = 32) with the fused exchange and the library's chunk order on every rank."""
    lat, rp, col, val = ti_problem((2 * P, 6, 16))
    planes = [lat.nx * q // P for q in range(P + 1)]
    bounds = [q * lat.rows_per_plane for q in planes]
    out = run_case(pkg, P, lat.n, rp, col, val, bounds, 64, R, SEED + P, want_v0=(R == 8))
    with pkg.KpmContext() as c1:  # P-invariance against one rank
        a, b = scale_factors(*gershgorin(rp, col, val))
        c1.set_matrix(rp, col, val, a, b)
        mu1, _ = c1.moments(64, R, SEED + P)
    err = float(np.max(np.abs(out[0]["mu"] - mu1)) / mu1[0])
    assert err <= TOL, err
    return dict(kernel=out[0]["kernel"], p_invariance=err)


def case_uneven(pkg, P):
    """Uneven row split of a TI lattice with random long-range couplings on rank 1: halo runs are
    scattered, some ranks cannot run the tiled / block-cache feeds -- all ranks agree on one
    variant (no hang), results oracle-exact."""
    n, rp, col, val = mixed_problem(P)
    w = np.arange(1, P + 1, dtype=float)
    bounds = [0] + [int(x) for x in np.round(np.cumsum(w) / w.sum() * n)]
    bounds[-1] = n
    out = run_case(pkg, P, n, rp, col, val, bounds, 48, 32, 23)
    return dict(kernel=out[0]["kernel"])


def case_mismatch(pkg):
    g = pkg.VirtualGroup(3)
    try:
        pkg.KpmContext(device=0, nranks=2, rank=0, vgroup=g)
        return dict(ok=False, error="group of 3 accepted for nranks = 2")
    except pkg.KpmError:
        return dict(rejected=True)
    finally:
        g.close()


def main():
    import faulthandler

    import paper_1410_5242_b200 as pkg

    if os.environ.get("VRANKS_DUMP_AFTER"):  # diagnostics: every thread's stack if a case hangs
        faulthandler.dump_traceback_later(float(os.environ["VRANKS_DUMP_AFTER"]), exit=True)

    kind = sys.argv[1]
    try:
        if kind == "ti":
            res = case_ti(pkg, int(sys.argv[2]), int(sys.argv[3]))
        elif kind == "uneven":
            res = case_uneven(pkg, int(sys.argv[2]))
        else:
            res = case_mismatch(pkg)
        res.setdefault("ok", True)
    except AssertionError as e:
        res = dict(ok=False, error=f"assertion: {e}")
    print("VRANKS_RESULT " + json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
