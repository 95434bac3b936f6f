"""CPU tests of the input generator (Eq. (1)) and the reference SELL-C-sigma / halo
builders in oracle/sell_ref.py."""
import numpy as np
import pytest

from oracle import sell_ref
from workloads.ti_lattice import (GAMMA, GAMMA5, ZERO_POTENTIAL, Lattice, bloch_energies, dense,
                                  generate_csr, gershgorin, scale_factors)


def test_clifford_algebra():
    """Gamma^a Hermitian, {Gamma^a, Gamma^b} = 2 delta_ab for a,b in 1..4."""
    for a in range(1, 5):
        assert np.array_equal(GAMMA[a], GAMMA[a].conj().T)
        for b in range(1, 5):
            ac = GAMMA[a] @ GAMMA[b] + GAMMA[b] @ GAMMA[a]
            assert np.array_equal(ac, 2 * np.eye(4) * (a == b))
        assert np.array_equal(GAMMA5 @ GAMMA[a] + GAMMA[a] @ GAMMA5, np.zeros((4, 4)))


@pytest.mark.parametrize("dims", [(8, 8, 8), (3, 5, 4), (4, 4, 3), (5, 3, 2)])
def test_structure(dims):
    """N = 4 Nx Ny Nz, Hermitian, N_nz = 13N - 16 Nx Ny ("~13N"),
    row lengths {11, 13}."""
    lat = Lattice(*dims)
    rp, col, val = generate_csr(lat)
    assert len(rp) - 1 == lat.n == 4 * np.prod(dims)
    assert rp[-1] == lat.nnz_expected()
    assert set(np.diff(rp).tolist()) <= {11, 13}
    h = dense(lat)
    assert np.array_equal(h, h.conj().T)
    # entries unique per row
    rows = np.repeat(np.arange(lat.n), np.diff(rp))
    assert len(set(zip(rows.tolist(), col.tolist()))) == len(col)


def test_paper_domain_size():
    """'a domain of size 100x100x40 ... a matrix with 1.6*10^6 rows'."""
    lat = Lattice(100, 100, 40)
    assert lat.n == 1_600_000
    assert abs(lat.nnz_expected() / lat.n - 13) < 0.1


def test_slab_generation_matches_full():
    lat = Lattice(6, 4, 5)
    rp, col, val = generate_csr(lat)
    r0, r1 = lat.row_of(2, 0, 0), lat.row_of(5, 0, 0)
    rps, cols, vals = generate_csr(lat, 2, 5)
    assert np.array_equal(rps, rp[r0 : r1 + 1] - rp[r0])
    assert np.array_equal(cols, col[rp[r0] : rp[r1]])
    assert np.array_equal(vals, val[rp[r0] : rp[r1]])


def test_bloch_spectrum_and_gershgorin():
    """Periodic V=0 lattice: dense spectrum == Bloch closed form; Gershgorin [-8, 8];
    the scaled spectrum lies in [-1+eps, 1-eps]."""
    lat = Lattice(4, 3, 5, potential=ZERO_POTENTIAL, periodic_z=True)
    e = np.linalg.eigvalsh(dense(lat))
    assert np.max(np.abs(np.sort(e) - np.sort(bloch_energies(lat)))) < 1e-12
    lo, hi = gershgorin(*generate_csr(lat))
    assert (lo, hi) == (-8.0, 8.0)
    lat2 = Lattice(6, 6, 5)
    rp, col, val = generate_csr(lat2)
    a, b = scale_factors(*gershgorin(rp, col, val))
    e2 = np.linalg.eigvalsh(dense(lat2))
    assert np.all(np.abs(a * (e2 - b)) <= 0.99 + 1e-12)


# ------------------------------------------------------------------ SELL reference ----
def _diag_first(rp, col, val):
    """CRS rows with each row's diagonal entry moved to the front (R18)."""
    oc, ov = [], []
    for i in range(len(rp) - 1):
        c, v = list(col[rp[i] : rp[i + 1]]), list(val[rp[i] : rp[i + 1]])
        if i in c:
            k = c.index(i)
            c = [c[k]] + c[:k] + c[k + 1 :]
            v = [v[k]] + v[:k] + v[k + 1 :]
        oc += c
        ov += v
    return np.array(oc), np.array(ov)


def test_sell1_is_crs():
    """C=1, sigma=1 -> the CRS sequence, each row's diagonal first."""
    lat = Lattice(3, 3, 3)
    rp, col, val = generate_csr(lat)
    s = sell_ref.build_sell(rp, col, val, C=1, sigma=1)
    ec, ev = _diag_first(rp, col, val)
    assert np.array_equal(s["val"], ev)
    assert np.array_equal(s["col"], ec.astype(np.int32))
    assert not np.array_equal(ec, col)  # the TI's diagonal is not first in CRS order
    # a row without a stored diagonal keeps its order
    rp2, col2, val2 = np.array([0, 2, 3]), np.array([1, 0, 0]), np.array([1 + 1j, 2, 3])
    s2 = sell_ref.build_sell(rp2, col2, val2, C=1, sigma=1)
    assert list(s2["col"]) == [0, 1, 0] and list(s2["val"]) == [2, 1 + 1j, 3]


@pytest.mark.parametrize("C,sigma", [(32, 1), (32, 64), (4, 8), (32, 128)])
def test_sell_round_trip_and_spmv(C, sigma):
    """CSR -> SELL -> entry set round trip; SELL SpMV == dense H x (padding inert)."""
    lat = Lattice(4, 3, 5)
    rp, col, val = generate_csr(lat)
    n = lat.n
    s = sell_ref.build_sell(rp, col, val, C=C, sigma=sigma)
    perm = s["perm"]
    ent = sell_ref.sell_to_csr_entries(s, n, C)
    rows = np.repeat(np.arange(n), np.diff(rp))
    invperm = np.empty(n, dtype=np.int64)
    invperm[perm] = np.arange(n)
    ref = sorted(zip(invperm[rows].tolist(), invperm[col].tolist(), val.tolist()))
    got = sorted((p, c, v) for p, c, v in ent if v != 0)
    assert got == ref
    # within-row order: the diagonal first, then the stored order
    _, ev = _diag_first(rp, col, val)
    p0 = invperm[7]
    c0 = p0 // C
    js = [int(s["cptr"][c0]) + j * C + p0 % C for j in range(rp[8] - rp[7])]
    assert np.array_equal(s["val"][js], ev[rp[7] : rp[8]])
    # SpMV in permuted numbering
    x = np.random.default_rng(0).normal(size=n) + 1j * np.random.default_rng(1).normal(size=n)
    xp = np.zeros(s["n_pad"], dtype=np.complex128)
    xp[:n] = x[perm]
    y = np.zeros(s["n_pad"], dtype=np.complex128)
    for c in range(len(s["clen"])):
        for j in range(int(s["clen"][c])):
            idx = int(s["cptr"][c]) + j * C + np.arange(C)
            y[c * C : (c + 1) * C] += s["val"][idx] * xp[s["col"][idx]]
    assert np.allclose(y[:n], (dense(lat) @ x)[perm], atol=1e-12)
    # descending length inside each sigma window
    lens = np.diff(rp)[perm]
    for w0 in range(0, n, max(sigma, 1)):
        seg = lens[w0 : w0 + sigma]
        assert np.all(np.diff(seg) <= 0)


def test_sell_ti_padding_is_exact_13n():
    """sigma=1, C=32, 8 | Nz: chunks of 8 sites align with z-columns, so the padded
    SELL storage is exactly 13 N slots."""
    lat = Lattice(8, 8, 8)
    rp, col, val = generate_csr(lat)
    s = sell_ref.build_sell(rp, col, val)
    assert int(s["cptr"][-1]) == 13 * lat.n


def test_halo_lists_xslab():
    """Row-block partition of an x-slab ordering: each rank's halo is the
    neighbouring x-planes, contiguous; periodic in x."""
    lat = Lattice(8, 3, 4)
    P = 4
    planes = lat.nx // P
    row_begins = np.array([p * planes * lat.rows_per_plane for p in range(P + 1)])
    cols_by_rank = []
    for p in range(P):
        rp, col, val = generate_csr(lat, p * planes, (p + 1) * planes)
        cols_by_rank.append(col)
        halo, owner = sell_ref.halo_list(col, row_begins[p], row_begins[p + 1], row_begins)
        left, right = (p - 1) % P, (p + 1) % P
        assert set(owner.tolist()) == {left, right}
        lp = lat.rows_per_plane
        assert np.array_equal(halo[owner == left], np.arange(row_begins[left + 1] - lp, row_begins[left + 1]))
        assert np.array_equal(halo[owner == right], np.arange(row_begins[right], row_begins[right] + lp))
    sl = sell_ref.send_lists(cols_by_rank, row_begins)
    assert len(sl) == 2 * P


def test_slab_bloch_spectrum_matches_dense():
    """tests/bloch_ref.py (open z, periodic x, y, V = 0) against dense eigvalsh."""
    import scipy.sparse as sp

    from bloch_ref import slab_energies

    for dims in ((6, 5, 4), (4, 7, 3)):
        lat = Lattice(*dims, potential=ZERO_POTENTIAL)
        rp, col, val = generate_csr(lat)
        e = np.sort(slab_energies(lat, rp, col, val, workers=2))
        ed = np.linalg.eigvalsh(sp.csr_matrix((val, col, rp), shape=(lat.n, lat.n)).toarray())
        assert np.max(np.abs(e - ed)) < 1e-12
