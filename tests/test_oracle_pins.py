"""Pins of the oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage it pins; together they are chosen so that a plausible
mistake in the oracle (dropped shift, wrong sign of the -w term, a transposed operand,
an off-by-one in the loop bound or the doubling, a wrong Z4 map) fails one of them.
"""
import os

import numpy as np
import pytest

from workloads.ti_lattice import (ZERO_POTENTIAL, Lattice, Superlattice, bloch_energies, dense,
                                  generate_csr, gershgorin, scale_factors, GAMMA5)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def cheb(n, x):
    """T_n(x) = cos(n arccos x) in extended precision (textbook closed form, |x| <= 1)."""
    x = np.asarray(x, dtype=np.longdouble)
    return np.cos(np.longdouble(n) * np.arccos(x))


def cheb_table(M, x):
    return np.array([cheb(n, x) for n in range(M)], dtype=np.float64)


def csr_from_dense(h):
    n = h.shape[0]
    rows, cols = np.nonzero(h)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp)
    return rp, cols.astype(np.int64), h[rows, cols]


# ---------------------------------------------------------------- Philox / Z4 ----
def test_philox_known_answers(oracle_lib):
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt"))
            if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(t, 16) for t in r]
        out = oracle_lib.philox4x32_10(v[0:4], v[4:6])
        assert [int(x) for x in out] == v[6:10]


def test_z4_start_vectors(oracle_lib):
    """|rand()> under reading R6: unit modulus, four phases, ~uniform, keyed by
    (global row, global column) so a sub-block equals the slice of the full block."""
    z = oracle_lib.z4_block(0, 4096, 0, 8, seed=0x14105242)
    assert np.all(np.abs(z) == 1.0)
    phases = np.round(np.angle(z) / (np.pi / 2)).astype(int) % 4
    counts = np.bincount(phases.ravel(), minlength=4)
    expected = z.size / 4
    chi2 = np.sum((counts - expected) ** 2 / expected)
    assert chi2 < 30.0  # 3 dof; p ~ 1e-6
    sub = oracle_lib.z4_block(1000, 24, 3, 2, seed=0x14105242)
    assert np.array_equal(sub, z[1000:1024, 3:5])
    # the top two bits of word 0 choose the phase {1, i, -1, -i}
    w = oracle_lib.philox4x32_10([5, 0, 7, 0], [0x14105242, 0])
    q = int(w[0]) >> 30
    assert z[5, 7] == [1, 1j, -1, -1j][q]
    # columns decorrelated: E[v_i^* v_j] ~ 0 for i != j
    c = (z.conj().T @ z) / z.shape[0]
    assert np.max(np.abs(c - np.eye(8))) < 0.1


# ---------------------------------------------------------------- closed forms ----
@pytest.mark.parametrize("mode", [0, 1])
def test_scalar_recurrence(oracle_lib, mode):
    """1x1 H~ = (x): m_n = T_n(x) |v|^2 (Eq. (3))."""
    h, a, b = 1.7, 0.45, 0.3
    x = a * (h - b)
    M = 200
    rp, col, val = np.array([0, 1]), np.array([0]), np.array([h + 0j])
    v0 = np.array([[0.6 - 0.8j]])
    eta = oracle_lib.kpm_eta_v0(rp, col, val, a, b, M, v0, mode=mode)
    mu, m = oracle_lib.eta_to_mu(eta)
    ref = cheb_table(M, x)
    assert np.max(np.abs(mu - ref)) < 1e-13
    # the eta themselves: eta_2k = T_k^2, eta_2k+1 = T_{k+1} T_k
    k = np.arange(M // 2)
    assert np.allclose(eta[0, 0::2].real, cheb_table(M // 2 + 1, x)[k] ** 2, atol=1e-14)
    assert np.allclose(eta[0, 1::2].real,
                       cheb_table(M // 2 + 1, x)[k + 1] * cheb_table(M // 2 + 1, x)[k], atol=1e-14)


@pytest.mark.parametrize("mode", [0, 1])
def test_diagonal_closed_form(oracle_lib, mode):
    """H = diag(lambda): mu_n = sum_i T_n(a(lambda_i - b)) for unit-modulus vectors,
    every column, any R (Eq. (3) + stochastic trace P:261 + doubling)."""
    rng = np.random.default_rng(1)
    n, M, R = 300, 128, 3
    lam = rng.uniform(-3.0, 5.0, n)
    a, b = scale_factors(lam.min(), lam.max())
    rp = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int64)
    eta = oracle_lib.kpm_eta(rp, col, lam.astype(np.complex128), a, b, M, R, seed=7, mode=mode)
    mu, m = oracle_lib.eta_to_mu(eta)
    ref = cheb_table(M, a * (lam - b)).sum(axis=1)
    assert np.max(np.abs(mu - ref)) / n < 1e-13
    for r in range(R):
        assert np.max(np.abs(m[r] - ref)) / n < 1e-13
    assert eta[0, 0].real == n  # eta_0 = N exactly for Z4 vectors


@pytest.mark.parametrize("pot", [ZERO_POTENTIAL, Superlattice(spacing=(3, 3), dot=(1, 2), depth=0.7)])
def test_dense_eigendecomposition_ti(oracle_lib, pot):
    """Whole oracle on a small TI Hamiltonian vs numpy.linalg.eigh (library routine):
    m_n^(r) = sum_i |<phi_i|nu_0^r>|^2 T_n(lambda~_i).  Complex Z4 vectors make a
    transposed (= conjugated) operand visible through the eigenvector weights."""
    lat = Lattice(4, 3, 5, potential=pot)
    h = dense(lat)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    M, R = 96, 3
    eta = oracle_lib.kpm_eta(rp, col, val, a, b, M, R, seed=11)
    mu, m = oracle_lib.eta_to_mu(eta)
    v = oracle_lib.z4_block(0, lat.n, 0, R, seed=11)
    lam, phi = np.linalg.eigh(h)
    w = np.abs(phi.conj().T @ v) ** 2  # (n, R)
    T = cheb_table(M, a * (lam - b))  # (M, n)
    ref = T @ w  # (M, R)
    assert np.max(np.abs(m.real - ref.T)) / lat.n < 1e-12
    assert np.max(np.abs(m.imag)) / lat.n < 1e-12
    # the transposed operand gives different moments here (so the test can see it)
    lam_t, phi_t = np.linalg.eigh(h.T)
    wt = np.abs(phi_t.conj().T @ v) ** 2
    assert np.max(np.abs((T @ wt) - ref)) / lat.n > 1e-6


def test_random_hermitian_sparse(oracle_lib):
    """Non-lattice Hermitian matrix with a nonzero shift b: dense eigh pin."""
    rng = np.random.default_rng(5)
    n = 120
    h = np.zeros((n, n), dtype=np.complex128)
    for _ in range(400):
        i, j = rng.integers(0, n, 2)
        z = rng.normal() + 1j * rng.normal()
        h[i, j] += z
        h[j, i] += np.conj(z)
    h += np.diag(rng.normal(3.0, 1.0, n))
    h = 0.5 * (h + h.conj().T)
    rp, col, val = csr_from_dense(h)
    a, b = scale_factors(*gershgorin(rp, col, val))
    assert abs(b) > 0.5
    M, R = 80, 2
    eta = oracle_lib.kpm_eta(rp, col, val, a, b, M, R, seed=3, col_begin=5)
    mu, m = oracle_lib.eta_to_mu(eta)
    v = oracle_lib.z4_block(0, n, 5, R, seed=3)
    lam, phi = np.linalg.eigh(h)
    ref = cheb_table(M, a * (lam - b)) @ (np.abs(phi.conj().T @ v) ** 2)
    assert np.max(np.abs(m.real - ref.T)) / n < 1e-12


def test_exact_trace_bloch(oracle_lib):
    """Full-basis trace (v0 = identity, summed): sum_r m_n^(r) = tr T_n(H~) with the
    Bloch closed-form spectrum of the V=0 periodic lattice; mu_0 = N."""
    lat = Lattice(4, 4, 3, potential=ZERO_POTENTIAL, periodic_z=True)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    M = 64
    eta = oracle_lib.kpm_eta_v0(rp, col, val, a, b, M, np.eye(lat.n, dtype=np.complex128))
    mu, m = oracle_lib.eta_to_mu(eta)
    tr = mu * lat.n
    ref = cheb_table(M, a * (bloch_energies(lat) - b)).sum(axis=1)
    assert tr[0] == lat.n
    assert np.max(np.abs(tr - ref)) / lat.n < 1e-12
    # chiral symmetry (Gamma^5 anticommutes with H at V=0, b=0): odd traces vanish
    assert b == 0.0
    assert np.max(np.abs(tr[1::2])) / lat.n < 1e-13


def test_chiral_pair_cancels_odd_moments(oracle_lib):
    """S = 1 (x) Gamma^5 anticommutes with H (V=0): for the start block {v, S v} the
    odd moments of the two columns cancel (off-diagonal gathers + sign of the -w term)."""
    lat = Lattice(4, 3, 4, potential=ZERO_POTENTIAL)
    h = dense(lat)
    S = np.kron(np.eye(lat.n // 4), GAMMA5)
    assert np.max(np.abs(S @ h + h @ S)) == 0.0
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    v = oracle_lib.z4_block(0, lat.n, 0, 1, seed=9)[:, 0]
    v0 = np.stack([v, S @ v], axis=1)
    eta = oracle_lib.kpm_eta_v0(rp, col, val, a, b, 64, v0)
    mu, m = oracle_lib.eta_to_mu(eta)
    assert np.max(np.abs(m[0, 1::2] + m[1, 1::2])) / lat.n < 1e-13
    assert np.max(np.abs(m[0, 0::2] - m[1, 0::2])) / lat.n < 1e-13
    assert np.max(np.abs(m[0, 1::2])) / lat.n > 1e-4  # not trivially zero


def test_chained_equals_fused(oracle_lib):
    """'The algorithm itself is untouched': Fig. 3 chain == Fig. 4 fused."""
    lat = Lattice(8, 8, 8)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    e0 = oracle_lib.kpm_eta(rp, col, val, a, b, 64, 2, seed=1, mode=0)
    e1 = oracle_lib.kpm_eta(rp, col, val, a, b, 64, 2, seed=1, mode=1)
    assert np.max(np.abs(e0 - e1)) <= 1e-13 * lat.n


def test_hermiticity_invariants(oracle_lib):
    """eta_2m real >= 0, Im eta_2m+1 at rounding level, |mu_n| <= mu_0 (spectrum of H~
    inside [-1, 1])."""
    lat = Lattice(8, 8, 8)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    eta = oracle_lib.kpm_eta(rp, col, val, a, b, 200, 4, seed=2)
    assert np.all(eta[:, 0::2].real >= 0) and np.all(eta[:, 0::2].imag == 0)
    assert np.max(np.abs(eta[:, 1::2].imag)) < 1e-12 * lat.n
    mu, _ = oracle_lib.eta_to_mu(eta)
    assert mu[0] == lat.n
    assert np.all(np.abs(mu) <= mu[0] * (1 + 1e-12))


def test_column_permutation_and_thread_invariance(oracle_lib):
    """Columns are independent and results are bitwise thread-count independent."""
    lat = Lattice(8, 8, 8)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    v0 = oracle_lib.z4_block(0, lat.n, 0, 3, seed=4)
    e = oracle_lib.kpm_eta_v0(rp, col, val, a, b, 32, v0, threads=1)
    ep = oracle_lib.kpm_eta_v0(rp, col, val, a, b, 32, v0[:, [2, 0, 1]], threads=4)
    assert np.array_equal(ep, e[[2, 0, 1]])


def test_rejects_bad_arguments(oracle_lib):
    rp, col, val = np.array([0, 1]), np.array([0]), np.array([1.0 + 0j])
    with pytest.raises(ValueError):
        oracle_lib.kpm_eta(rp, col, val, 0.5, 0.0, 7, 1, seed=0)  # odd M
    with pytest.raises(ValueError):
        oracle_lib.kpm_eta(rp, col, val, -0.5, 0.0, 8, 1, seed=0)  # a <= 0
    with pytest.raises(ValueError):
        oracle_lib.kpm_eta(rp, np.array([3]), val, 0.5, 0.0, 8, 1, seed=0)  # column range
