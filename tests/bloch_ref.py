"""Exact spectra of the V = 0 TI lattice for full-size pins (SURVEY §8(c) "partial Bloch").

H is translation invariant in x and y (periodic, V = 0), so it is block-diagonal in
(kx, ky) with 4Nz x 4Nz blocks H(k) = sum_D H_D exp(i k.D), H_D read off the CSR rows of
the site column (x, y) = (0, 0).  Built from the generated matrix itself (no KPM
arithmetic); pinned against a dense eigendecomposition in test_workloads_and_sell_ref.py."""
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np


def hopping_blocks(lat, rp, col, val):
    nb = 4 * lat.nz
    blocks = {}
    for r in range(nb):
        for e in range(rp[r], rp[r + 1]):
            site, o = divmod(int(col[e]), 4)
            z, xy = site % lat.nz, site // lat.nz
            x, y = divmod(xy, lat.ny)
            dx = x if x <= lat.nx // 2 else x - lat.nx
            dy = y if y <= lat.ny // 2 else y - lat.ny
            blocks.setdefault((dx, dy), np.zeros((nb, nb), complex))[r, 4 * z + o] += val[e]
    return blocks


def _init_worker():
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)  # one BLAS thread per process: the processes are the parallelism


def _row(args):
    blocks, kx, ky = args
    hk = sum(B[None] * np.exp(1j * (kx * dx + ky[:, None, None] * dy)) for (dx, dy), B in blocks.items())
    return np.linalg.eigvalsh(hk).ravel()


def slab_energies(lat, rp, col, val, workers=None):
    """All N eigenvalues of H (V = 0, periodic x, y, any z boundary)."""
    blocks = hopping_blocks(lat, rp, col, val)
    ky = 2 * np.pi * np.arange(lat.ny) / lat.ny
    jobs = [(blocks, 2 * np.pi * i / lat.nx, ky) for i in range(lat.nx)]
    workers = workers or min(32, os.cpu_count() or 1)
    if workers == 1 or lat.nx < 4:
        return np.concatenate([_row(j) for j in jobs])
    import multiprocessing as mp

    with ProcessPoolExecutor(workers, mp_context=mp.get_context("spawn"), initializer=_init_worker) as ex:
        return np.concatenate(list(ex.map(_row, jobs, chunksize=max(1, lat.nx // (4 * workers)))))


def cheb_moments(x, M):
    """tr T_n(x) and sum T_n(x)^2 over the eigenvalues x (|x| < 1), n < M, by the three-term
    recurrence in float64 (|T_n| <= 1; error ~ n eps per term)."""
    t0, t1 = np.ones_like(x), x.copy()
    tr, sq = np.zeros(M), np.zeros(M)
    for n in range(M):
        tr[n], sq[n] = t0.sum(), (t0 * t0).sum()
        t0, t1 = t1, 2 * x * t1 - t0
    return tr, sq
