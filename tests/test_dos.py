"""Jackson-kernel DOS reconstruction (north_star item 5): the oracle's
`dos` pinned by closed forms, an independent construction of the Jackson kernel, exact
Gauss-Chebyshev normalisation and the dense eigenvalue histogram; the library's host
`kpm_dos` (CPU, no GPU needed) against the oracle."""
import numpy as np
import pytest

import oracle
from workloads.ti_lattice import Lattice, dense, generate_csr, gershgorin, scale_factors


@pytest.mark.parametrize("M", [2, 10, 64, 1000])
def test_jackson_is_autocorrelation(M):
    """g_n = sum_nu a_nu a_{nu+n} / sum a_nu^2 with a_nu = sin(pi (nu+1)/(M+1)): the kernel's
    construction as the optimal positive kernel, computed independently of the closed form."""
    a = np.sin(np.pi * (np.arange(M) + 1) / (M + 1))
    ac = np.array([np.dot(a[: M - n], a[n:]) for n in range(M)]) / np.dot(a, a)
    assert np.max(np.abs(oracle.jackson(M) - ac)) < 1e-14
    assert oracle.jackson(M)[0] == pytest.approx(1.0, abs=1e-15)


def test_flat_moments_closed_form():
    """mu = (N, 0, ...): rho~(x) = N / (pi sqrt(1 - x^2)), in E units times a."""
    N, a, b = 37.0, 0.2, -1.5
    mu = np.zeros(40)
    mu[0] = N
    for kern in ("none", "jackson"):
        E, rho = oracle.dos(mu, a, b, K=101, kernel=kern)
        x = a * (E - b)
        assert np.allclose(rho, a * N / (np.pi * np.sqrt(1 - x * x)), rtol=1e-13)


def test_normalisation_exact_quadrature():
    """At K > M Chebyshev nodes, pi/K sum_k rho~(x_k) sqrt(1-x_k^2) = mu_0 exactly (Gauss-Chebyshev)."""
    rng = np.random.default_rng(3)
    mu = rng.normal(size=60)
    mu[0] = 123.0
    a, b = 0.5, 0.1
    E, rho = oracle.dos(mu, a, b, K=200)
    x = a * (E - b)
    total = np.pi / len(x) * np.sum(rho / a * np.sqrt(1 - x * x))
    assert total == pytest.approx(123.0, rel=1e-13)


def test_delta_positive_and_centred():
    """One eigenvalue x0: mu_n = T_n(x0).  Jackson keeps rho~ >= 0 (the kernel's purpose) and
    the broadened peak integrates to 1 with its maximum next to x0."""
    x0, M = 0.3, 400
    mu = np.cos(np.arange(M) * np.arccos(x0))
    E, rho = oracle.dos(mu, 1.0, 0.0, K=4000)
    assert np.min(rho) > -1e-10
    x = E
    assert np.pi / len(x) * np.sum(rho * np.sqrt(1 - x * x)) == pytest.approx(1.0, rel=1e-12)
    assert abs(x[np.argmax(rho)] - x0) < 0.01
    E2, rho2 = oracle.dos(mu, 1.0, 0.0, K=4000, kernel="none")
    assert np.min(rho2) < -1.0  # Gibbs oscillations without the kernel


def test_dense_histogram_ti():
    """DOS of the 4x4x4 TI (N = 256) from exact-trace moments vs the dense eigenvalue
    histogram on 16 bins (SPEC acceptance criterion 4: <= 5% of N per bin)."""
    lat = Lattice(4, 4, 4)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    M = 1000
    eta = oracle.kpm_eta_v0(rp, col, val, a, b, M, np.eye(lat.n, dtype=np.complex128))
    mu, _ = oracle.eta_to_mu(eta)
    mu = mu * lat.n  # exact trace: sum over the basis
    lam = np.linalg.eigvalsh(dense(lat))
    edges = np.linspace(b - 1 / a, b + 1 / a, 17)
    fine = np.linspace(edges[0], edges[-1], 64001)[1:-1]
    E, rho = oracle.dos(mu, a, b, energies=fine)
    dE = fine[1] - fine[0]
    for lo, hi in zip(edges[:-1], edges[1:]):
        sel = (fine >= lo) & (fine < hi)
        kpm_count = rho[sel].sum() * dE
        exact = np.sum((lam >= lo) & (lam < hi))
        assert abs(kpm_count - exact) <= 0.05 * lat.n, (lo, hi, kpm_count, exact)
    assert rho.sum() * dE == pytest.approx(lat.n, rel=1e-3)


@pytest.fixture(scope="module")
def pkg():
    from paper_1410_5242_b200 import build

    build.build()
    import paper_1410_5242_b200 as p

    return p


@pytest.mark.parametrize("kernel", ["jackson", "none"])
def test_library_dos_matches_oracle(pkg, kernel):
    rng = np.random.default_rng(7)
    mu = rng.normal(size=500) * np.exp(-np.arange(500) / 200)
    mu[0] = 1e6
    a, b = 0.12375, 0.25
    E1, r1 = pkg.dos(mu, a, b, K=3000, kernel=kernel)
    E2, r2 = oracle.dos(mu, a, b, K=3000, kernel=kernel)
    assert np.array_equal(E1, E2) or np.max(np.abs(E1 - E2)) < 1e-12
    assert np.max(np.abs(r1 - r2)) <= 1e-11 * np.max(np.abs(r2))
    en = np.linspace(-9, 9, 777)  # includes points outside [b - 1/a, b + 1/a]
    E3, r3 = pkg.dos(mu, a, b, energies=en, kernel=kernel)
    inside = np.abs(a * (en - b)) < 1
    E4, r4 = oracle.dos(mu, a, b, energies=en[inside], kernel=kernel)
    assert np.max(np.abs(r3[inside] - r4)) <= 1e-11 * np.max(np.abs(r4))
    assert np.all(r3[~inside] == 0)
