"""GPU parity: the CUDA path through the C ABI vs the oracle, element by element on the
same seeded inputs (north_star gate: max_n |mu_gpu - mu_oracle| / mu_0 <= 1e-10, and per
column max_n |eta_gpu - eta_oracle| / eta_0 <= 1e-10)."""
import numpy as np
import pytest

import oracle
from oracle import sell_ref
from workloads.ti_lattice import (SEED, ZERO_POTENTIAL, Lattice, bloch_energies, gershgorin, generate_csr,
                                  scale_factors)

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1410_5242_b200 import build

    build.build()
    import paper_1410_5242_b200 as p

    return p


def problem(dims, potential=None, periodic_z=False):
    lat = Lattice(*dims, periodic_z=periodic_z) if potential is None else Lattice(*dims, potential=potential,
                                                                                  periodic_z=periodic_z)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    return lat, rp, col, val, a, b


def ref_sell(rp, col, val, **kw):
    """The product's SELL contract: the layout of the numpy reference builder (R18)."""
    return sell_ref.build_sell(rp, col, val, **kw)


def check(eta_g, mu_g, eta_o, cols=None):
    if cols is not None:
        eta_g = eta_g[cols]
    eta0 = eta_o[:, :1].real
    col_err = np.max(np.abs(eta_g - eta_o) / eta0)
    assert col_err <= TOL, col_err
    if cols is None:
        mu_o, _ = oracle.eta_to_mu(eta_o)
        assert np.max(np.abs(mu_g - mu_o)) / mu_o[0] <= TOL
    return col_err


@pytest.mark.parametrize("R", [1, 2, 4, 8, 16, 32])
def test_c1_all_widths(pkg, R):
    lat, rp, col, val, a, b = problem((8, 8, 8))
    M = 64
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, eta = ctx.moments(M, R, SEED)
    eta_o = oracle.kpm_eta(rp, col, val, a, b, M, R, SEED)
    check(eta, mu, eta_o)
    assert mu[0] == lat.n  # Z4 vectors: eta_0 = N exactly


@pytest.mark.parametrize("R", [3, 5, 33, 40])
def test_ragged_widths_and_batches(pkg, R):
    """Non-power-of-two widths pad to the next kernel width; R > 32 runs in blocks of 32
    whose Philox columns continue the global column numbering."""
    lat, rp, col, val, a, b = problem((6, 5, 7))  # N = 840: ragged last chunk (840 = 26*32 + 8)
    M = 40
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, eta = ctx.moments(M, R, SEED + 1)
    eta_o = oracle.kpm_eta(rp, col, val, a, b, M, R, SEED + 1)
    check(eta, mu, eta_o)


@pytest.mark.parametrize("sigma", [1, 64])
def test_zero_potential_and_sigma(pkg, sigma):
    lat, rp, col, val, a, b = problem((5, 4, 9), potential=ZERO_POTENTIAL)
    M, R = 100, 8
    with pkg.KpmContext(sell_sigma=sigma) as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, eta = ctx.moments(M, R, 77)
        s = ctx.export_sell()
    eta_o = oracle.kpm_eta(rp, col, val, a, b, M, R, 77)
    check(eta, mu, eta_o)
    ref = ref_sell(rp, col, val, C=32, sigma=sigma)
    assert np.array_equal(s["cptr"], ref["cptr"])
    assert np.array_equal(s["col"], ref["col"])
    assert np.array_equal(s["val"], ref["val"])
    assert np.array_equal(s["perm"], ref["perm"])


def test_sell_bit_exact_c1(pkg):
    lat, rp, col, val, a, b = problem((8, 8, 8))
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        s = ctx.export_sell()
    ref = ref_sell(rp, col, val)
    for k in ("cptr", "col", "val", "perm"):
        assert np.array_equal(s[k], ref[k]), k
    assert s["cptr"][-1] == 13 * lat.n


def test_exact_trace_bloch_v0(pkg):
    """kpm_moments_v0 with the full basis (R = N, 20 blocks of 32): sum_r m_n = tr T_n(H~)
    from the Bloch closed form (periodic V=0 lattice)."""
    lat, rp, col, val, a, b = problem((4, 4, 5), potential=ZERO_POTENTIAL, periodic_z=True)
    M = 64
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, eta = ctx.moments_v0(M, np.eye(lat.n, dtype=np.complex128))
    tr = mu * lat.n
    x = a * (bloch_energies(lat) - b)
    ref = np.array([np.cos(n * np.arccos(np.clip(x, -1, 1))).sum() for n in range(M)])
    assert np.max(np.abs(tr - ref)) / lat.n < 1e-12


def test_explicit_v0_matches_oracle(pkg):
    lat, rp, col, val, a, b = problem((4, 3, 6))
    rng = np.random.default_rng(0)
    v0 = rng.normal(size=(lat.n, 3)) + 1j * rng.normal(size=(lat.n, 3))
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, eta = ctx.moments_v0(50, v0)
    eta_o = oracle.kpm_eta_v0(rp, col, val, a, b, 50, v0)
    check(eta, mu, eta_o)


def test_deterministic(pkg):
    lat, rp, col, val, a, b = problem((8, 8, 8))
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu1, e1 = ctx.moments(64, 16, 5)
        mu2, e2 = ctx.moments(64, 16, 5)
    assert np.array_equal(e1, e2) and np.array_equal(mu1, mu2)


def test_errors(pkg):
    lat, rp, col, val, a, b = problem((3, 3, 2))
    with pkg.KpmContext() as ctx:
        with pytest.raises(pkg.KpmError) as ei:
            ctx.moments(8, 1, 0)
        assert ei.value.status == pkg.KPM_ESTATE
        with pytest.raises(pkg.KpmError) as ei:
            ctx.set_matrix(rp, col, val, -1.0, b)
        assert ei.value.status == pkg.KPM_EINVAL
        bad = col.copy()
        bad[3] = lat.n
        with pytest.raises(pkg.KpmError) as ei:
            ctx.set_matrix(rp, bad, val, a, b)
        assert ei.value.status == pkg.KPM_ERANGE
        ctx.set_matrix(rp, col, val, a, b)
        with pytest.raises(pkg.KpmError) as ei:
            ctx.moments(7, 1, 0)
        assert ei.value.status == pkg.KPM_EINVAL
        # a too large: spectrum leaves [-1, 1] -> WDIVERGED warning, results written
        ctx.set_matrix(rp, col, val, 3 * a, b)
        mu, _ = ctx.moments(64, 2, 0, allow_warning=True)
        assert ctx.last_status == pkg.KPM_WDIVERGED
        z = np.zeros((lat.n, 1), dtype=np.complex128)
        with pytest.raises(pkg.KpmError) as ei:
            ctx.moments_v0(8, z, allow=())
        assert ei.value.status == pkg.KPM_EZERONORM


def test_c2_full(pkg):
    """Config 2 (64x64x32, M=1000, R=8) in the bench launch configuration; the oracle
    computes the sampled columns 0 and 7 in full."""
    lat, rp, col, val, a, b = problem((64, 64, 32))
    M, R = 1000, 8
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, eta = ctx.moments(M, R, SEED)
    for c in (0, 7):
        eta_o = oracle.kpm_eta(rp, col, val, a, b, M, 1, SEED, col_begin=c)
        check(eta[c : c + 1], None, eta_o, cols=[0])
    assert mu[0] == lat.n and np.all(np.abs(mu) <= mu[0])


def test_c3_sampled_columns(pkg):
    """Config 3 (200x100x40, R=32) at M=200: sampled columns 0 and 31 against the oracle;
    mu_0 = N and |mu_n| <= mu_0 at full size."""
    lat, rp, col, val, a, b = problem((200, 100, 40))
    M, R = 200, 32
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, eta = ctx.moments(M, R, SEED)
    for c in (0, 31):
        eta_o = oracle.kpm_eta(rp, col, val, a, b, M, 1, SEED, col_begin=c)
        check(eta[c : c + 1], None, eta_o, cols=[0])
    assert mu[0] == lat.n and np.all(np.abs(mu) <= mu[0])


def test_dos_pipeline_c1(pkg):
    """GPU moments -> library Jackson DOS == oracle moments -> oracle DOS; integrates to N."""
    lat, rp, col, val, a, b = problem((8, 8, 8))
    M, R = 256, 16
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, _ = ctx.moments(M, R, SEED)
    mu_o, _ = oracle.eta_to_mu(oracle.kpm_eta(rp, col, val, a, b, M, R, SEED))
    E, rho = pkg.dos(mu, a, b, K=1024)
    E_o, rho_o = oracle.dos(mu_o, a, b, K=1024)
    assert np.max(np.abs(rho - rho_o)) <= 1e-10 * np.max(rho_o)
    x = a * (E - b)
    assert np.pi / len(x) * np.sum(rho / a * np.sqrt(1 - x * x)) == pytest.approx(lat.n, rel=1e-12)


@pytest.mark.parametrize("R", [1, 2, 4, 8, 16, 32])
def test_every_kernel_variant(pkg, R, monkeypatch):
    """Each aug_spmmv variant of a width (tiled / staged / direct feeds, lane maps, unrolls;
    KPM_VARIANT) against the oracle, on a lattice with a ragged last chunk."""
    lat, rp, col, val, a, b = problem((5, 6, 9))
    M = 48
    eta_o = oracle.kpm_eta(rp, col, val, a, b, M, R, SEED)
    seen = set()
    for v in range(16):
        want = pkg.variant_name(R, v)
        if want is None:
            break
        monkeypatch.setenv("KPM_VARIANT", str(v))
        with pkg.KpmContext() as ctx:
            ctx.set_matrix(rp, col, val, a, b)
            mu, eta = ctx.moments(M, R, SEED)
            name = ctx.last_kernel()
        # only a variant whose plan cannot fit this matrix (block cache, staged) falls back
        assert name == want or ".bc." in want or want.startswith("staged"), (want, name)
        seen.add(name)
        check(eta, mu, eta_o)
    assert len(seen) >= 2


def test_chunk_order_hint(pkg):
    """kpm_set_chunk_order changes only the rounding of the eta sums; bad orders rejected."""
    from workloads.ti_lattice import chunk_order_yband

    lat, rp, col, val, a, b = problem((6, 10, 16))
    M, R = 64, 32
    eta_o = oracle.kpm_eta(rp, col, val, a, b, M, R, SEED)
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        ctx.set_chunk_order(chunk_order_yband(lat, 0, lat.nx, 3))
        mu, eta = ctx.moments(M, R, SEED)
        check(eta, mu, eta_o)
        mu2, _ = ctx.moments(M, R, SEED)
        assert np.array_equal(mu, mu2)
        with pytest.raises(pkg.KpmError):
            ctx.set_chunk_order(np.zeros(ctx.sell_info().n_chunks, dtype=np.int64))
        ctx.set_chunk_order(None)
        mu3, eta3 = ctx.moments(M, R, SEED)
        check(eta3, mu3, eta_o)


@pytest.mark.parametrize("dims", [(8, 8, 8), (6, 5, 7), (10, 9, 16)])
def test_device_build(pkg, dims):
    """kpm_set_matrix from a CSR already on the GPU (KPM_MEM_DEVICE): the device SELL and
    tile-plan builder gives the reference SELL bit for bit and oracle-exact moments."""
    import torch

    from workloads.ti_lattice import generate_csr_torch

    lat, rp, col, val, a, b = problem(dims)
    rp_d, col_d, val_d = generate_csr_torch(lat, device="cuda")
    M = 48
    for R in (4, 32):
        with pkg.KpmContext() as ctx:
            ctx.set_matrix(rp_d, col_d, val_d, a, b, n_global=lat.n, mem=pkg.KPM_MEM_DEVICE)
            s = ctx.export_sell()
            mu, eta = ctx.moments(M, R, SEED)
            assert ctx.last_kernel().startswith("tiled")
        ref = ref_sell(rp, col, val)
        for k in ("cptr", "col", "val", "perm"):
            assert np.array_equal(s[k], ref[k]), k
        check(eta, mu, oracle.kpm_eta(rp, col, val, a, b, M, R, SEED))
    torch.cuda.synchronize()


def test_device_build_errors(pkg):
    import torch

    lat, rp, col, val, a, b = problem((4, 3, 8))
    bad = torch.as_tensor(col, device="cuda").clone()
    bad[5] = lat.n + 3
    with pkg.KpmContext() as ctx:
        with pytest.raises(pkg.KpmError) as ei:
            ctx.set_matrix(torch.as_tensor(rp, device="cuda"), bad, torch.as_tensor(val, device="cuda"), a, b,
                           n_global=lat.n, mem=pkg.KPM_MEM_DEVICE)
        assert ei.value.status == pkg.KPM_ERANGE


def _rows_without_diagonal():
    """TI lattice (10x9x16) whose diagonal entry is dropped in every third row (H_ii = 0 not
    stored) and split into two entries in every seventh row: the diagonal-first SELL order
    (R18) then meets rows where entry 0 is not the own row, rows where it is, and
    duplicates, inside the same warps of the tiled kernel."""
    lat = Lattice(10, 9, 16)
    rp, col, val = generate_csr(lat)
    rows, cols, vals = [], [], []
    for i in range(lat.n):
        c, v = col[rp[i] : rp[i + 1]], val[rp[i] : rp[i + 1]]
        for cj, vj in zip(c, v):
            if cj == i and i % 3 == 0:
                continue
            if cj == i and i % 7 == 0:
                rows += [i, i]
                cols += [cj, cj]
                vals += [0.25 * vj, 0.75 * vj]
                continue
            rows.append(i)
            cols.append(cj)
            vals.append(vj)
    rows = np.array(rows)
    rp2 = np.zeros(lat.n + 1, dtype=np.int64)
    np.add.at(rp2, rows + 1, 1)
    return lat, np.cumsum(rp2), np.array(cols, dtype=np.int64), np.array(vals, dtype=np.complex128)


@pytest.mark.parametrize("R", [2, 8, 16, 32])
def test_rows_without_diagonal(pkg, R):
    lat, rp, col, val = _rows_without_diagonal()
    a, b = scale_factors(*gershgorin(rp, col, val))
    import torch

    M = 64
    eta_o = oracle.kpm_eta(rp, col, val, a, b, M, R, SEED)
    ref = ref_sell(rp, col, val)
    for dev in (False, True):  # host builder, device builder
        with pkg.KpmContext() as ctx:
            if dev:
                ctx.set_matrix(torch.as_tensor(rp, device="cuda"), torch.as_tensor(col, device="cuda"),
                               torch.as_tensor(val, device="cuda"), a, b, n_global=lat.n, mem=pkg.KPM_MEM_DEVICE)
            else:
                ctx.set_matrix(rp, col, val, a, b)
            mu, eta = ctx.moments(M, R, SEED)
            assert ctx.last_kernel().startswith("tiled")
            s = ctx.export_sell()
        check(eta, mu, eta_o)
        assert np.array_equal(s["col"], ref["col"]) and np.array_equal(s["val"], ref["val"])


@pytest.mark.parametrize("ordered", [False, True])
@pytest.mark.parametrize("R,dims,name,ctas", [(32, (40, 20, 32), "tiled.bc.lpr8.u4", 1),
                                             (16, (80, 12, 32), "tiled.bc.lpr8.u4.wr", 2),
                                             (16, (80, 12, 32), "tiled.bc.lpr4.u4.wr", 2),
                                             (8, (120, 8, 32), "tiled.bc.lpr4.u4.wr", 3)])
def test_block_cache_feed(pkg, monkeypatch, ordered, R, dims, name, ctas):
    """Block-cache feed (tiled.bc): per-CTA pools of 32-row V blocks reused across tiles.  On
    lattices with more z-block lines than CTAs (one lock-stepped round + a storage-order tail),
    with and without the y-line order: oracle-exact, and the variant really ran."""
    import torch

    from workloads.ti_lattice import chunk_order_ylines

    lat, rp, col, val, a, b = problem(dims)
    M = 24
    idx = [pkg.variant_name(R, v) for v in range(16)].index(name)
    monkeypatch.setenv("KPM_VARIANT", str(idx))
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        if ordered:
            sms = torch.cuda.get_device_properties(0).multi_processor_count
            ctx.set_chunk_order(chunk_order_ylines(lat, ctas * sms))
        mu, eta = ctx.moments(M, R, SEED)
        assert ctx.last_kernel() == name
    check(eta, mu, oracle.kpm_eta(rp, col, val, a, b, M, R, SEED))


def _full_orbital_blocks(dims, xblocks=True, seed=5):
    """The TI plus random complex Hermitian couplings filling its on-site (and, xblocks, its +-x)
    4x4 orbital blocks: the same 32-row block neighbourhoods as the TI, so the block-cache plan
    can fit, but rows of 14-16 (18-20) entries (4-entry batches plus remainders, wider val / lcol
    blocks per stage) instead of the TI's 11-13."""
    import scipy.sparse as sp

    lat, rp, col, val, _, _ = problem(dims)
    rows = np.repeat(np.arange(lat.n), np.diff(rp))
    sites = np.unique(np.stack([rows // 4, col // 4], 1), axis=0)
    ns, nx_stride = lat.n // 4, dims[1] * dims[2]  # x is the slowest site index (R15)
    d = (sites[:, 1] - sites[:, 0]) % ns
    sites = sites[(d == 0) | (xblocks & ((d == nx_stride) | (d == ns - nx_stride)))]  # blocks filled
    o = np.arange(4)
    r = (sites[:, :1, None] * 4 + o[None, :, None] + 0 * o[None, None, :]).reshape(-1)
    c = (sites[:, 1:, None] * 4 + 0 * o[None, :, None] + o[None, None, :]).reshape(-1)
    rng = np.random.default_rng(seed)
    z = rng.normal(size=len(r)) + 1j * rng.normal(size=len(r))
    h = sp.coo_matrix((z, (r, c)), shape=(lat.n, lat.n)).tocsr()
    h = (h + h.conj().T + sp.csr_matrix((val, col, rp), shape=(lat.n, lat.n))).tocsr()
    h.sort_indices()
    rp2, col2, val2 = h.indptr.astype(np.int64), h.indices.astype(np.int64), h.data.astype(np.complex128)
    a, b = scale_factors(*gershgorin(rp2, col2, val2))
    return lat, rp2, col2, val2, a, b


@pytest.mark.parametrize("R,name", [(32, "tiled.bc.lpr8.u4"), (16, "tiled.bc.lpr8.u4.wr")])
def test_block_cache_wide_rows(pkg, monkeypatch, R, name):
    """Rows wider than the TI's (14-16 entries) on the block-cache feed (the R = 16 / 32
    defaults): oracle-exact, and the named variant really ran.  (16 is the widest chunk whose
    stages leave the 5 S = 10 pool slots the plan needs at both widths.)"""
    lat, rp, col, val, a, b = _full_orbital_blocks((24, 10, 32), xblocks=False)
    assert np.diff(rp).max() > 13
    idx = [pkg.variant_name(R, v) for v in range(16)].index(name)
    monkeypatch.setenv("KPM_VARIANT", str(idx))
    M = 24
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, eta = ctx.moments(M, R, SEED)
        assert ctx.last_kernel() == name
    check(eta, mu, oracle.kpm_eta(rp, col, val, a, b, M, R, SEED))


@pytest.mark.parametrize("R", [1, 8, 32])
def test_irregular_matrix_fallback(pkg, R):
    """A random Hermitian matrix with empty rows, wide rows (up to ~200 entries) and scattered
    columns: no tile plan fits (too many runs / rows per chunk), so the default selection falls
    back to the direct feed -- still oracle-exact."""
    rng = np.random.default_rng(11)
    n = 3000
    rows, cols = [], []
    for i in range(n):
        k = 0 if i % 97 == 0 else int(rng.integers(1, 200 if i % 13 == 0 else 12))
        rows += [i] * k
        cols += rng.integers(0, n, k).tolist()
    rows, cols = np.array(rows), np.array(cols)
    keep = (rows % 97 != 0) & (cols % 97 != 0)  # rows (and columns) 0, 97, ... stay empty
    rows, cols = rows[keep], cols[keep]
    z = rng.normal(size=len(rows)) + 1j * rng.normal(size=len(rows))
    import scipy.sparse as sp

    h = sp.coo_matrix((z, (rows, cols)), shape=(n, n)).tocsr()
    h = (h + h.conj().T).tocsr()
    h.sort_indices()
    rp, col, val = h.indptr.astype(np.int64), h.indices.astype(np.int64), h.data.astype(np.complex128)
    a, b = scale_factors(*gershgorin(rp, col, val))
    M = 40
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, eta = ctx.moments(M, R, SEED)
        assert ctx.last_kernel().startswith("direct")
    check(eta, mu, oracle.kpm_eta(rp, col, val, a, b, M, R, SEED))


@pytest.mark.parametrize("stage", ["naive", "aug_spmv", "aug_spmmv"])
def test_optimisation_stages(pkg, stage):
    """The three stages of Figs. 3-5 give the same moments (P:89-90 'the algorithm itself is
    untouched'), each against the oracle."""
    lat, rp, col, val, a, b = problem((6, 5, 8))
    M, R = 40, 5
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, eta = ctx.moments_stage(stage, M, R, SEED)
    check(eta, mu, oracle.kpm_eta(rp, col, val, a, b, M, R, SEED, mode=oracle.CHAINED))


@pytest.mark.parametrize("sigma", [1, 64])
def test_host_builder_forced(pkg, sigma, monkeypatch):
    """KPM_HOST_BUILD=1 keeps the multithreaded host builder (the default for host input with
    sigma = 1 is the device builder after one H2D copy): both give the reference SELL."""
    monkeypatch.setenv("KPM_HOST_BUILD", "1")
    lat, rp, col, val, a, b = problem((6, 5, 8))
    with pkg.KpmContext(sell_sigma=sigma) as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        s = ctx.export_sell()
        mu, eta = ctx.moments(40, 8, SEED)
    ref = ref_sell(rp, col, val, C=32, sigma=sigma)
    for k in ("cptr", "col", "val", "perm"):
        assert np.array_equal(s[k], ref[k]), k
    check(eta, mu, oracle.kpm_eta(rp, col, val, a, b, 40, 8, SEED))


@pytest.mark.parametrize("R", [1, 4, 8, 16, 32])
@pytest.mark.parametrize("kind", ["spmmv", "aug_nodot", "aug"])
def test_analysis_kernels(pkg, kind, R):
    """kpm_sweep_kernel (the paper's three kernels of the bottleneck analysis):
    W = H V for the plain SpMMV; W = 2a(H - b)V after one augmented sweep from W = 0; after
    two, W = fma(2a, u, -W1) = the rounding residual of W1 (|.| <= ulp/2), and after three
    round(2a u - residual) = W1 exactly.  V = the oracle's Z4 block;
    H V by scipy.sparse (a library product, not the kernel's arithmetic)."""
    import scipy.sparse as sp

    lat, rp, col, val, a, b = problem((6, 5, 7))  # ragged last chunk
    V = oracle.z4_block(0, lat.n, 0, R, SEED)
    HV = sp.csr_matrix((val, col, rp), shape=(lat.n, lat.n)) @ V
    want = HV if kind == "spmmv" else 2 * a * (HV - b * V)
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        ms, w1 = ctx.sweep_kernel(kind, R, SEED, n_sweeps=1, want_w=True)
        assert ms > 0
        assert ctx.last_kernel().endswith({"spmmv": ".spmmv", "aug_nodot": ".nodot", "aug": ""}[kind])
        _, w2 = ctx.sweep_kernel(kind, R, SEED, n_sweeps=2, want_w=True)
        _, w3 = ctx.sweep_kernel(kind, R, SEED, n_sweeps=3, want_w=True)
    scale = np.max(np.abs(want))
    assert np.max(np.abs(w1 - want)) <= 1e-13 * scale
    if kind == "spmmv":
        assert np.array_equal(w2, w1) and np.array_equal(w3, w1)
    else:
        assert np.max(np.abs(w2)) <= 2.0 ** -52 * scale and np.array_equal(w3, w1)


def test_analysis_kernel_errors(pkg):
    lat, rp, col, val, a, b = problem((4, 4, 4))
    with pkg.KpmContext() as ctx:
        with pytest.raises(pkg.KpmError) as e:
            ctx.sweep_kernel("spmmv", 8, SEED)
        assert e.value.status == pkg.KPM_ESTATE
        ctx.set_matrix(rp, col, val, a, b)
        for R in (0, 3, 64):
            with pytest.raises(pkg.KpmError) as e:
                ctx.sweep_kernel("aug", R, SEED)
            assert e.value.status == pkg.KPM_EINVAL
        with pytest.raises(pkg.KpmError) as e:
            ctx.sweep_kernel("aug", 8, SEED, n_sweeps=0)
        assert e.value.status == pkg.KPM_EINVAL
        assert ctx.lib.kpm_sweep_kernel(ctx.h, 7, 8, SEED, 1, None, None) == pkg.KPM_EINVAL  # unknown kind
        mu, _ = ctx.moments(16, 4, SEED)  # context still usable
        assert mu[0] == lat.n


def test_c3_full_size_partial_bloch(pkg):
    """Full C3 size (200x100x40, N = 3.2M) at V = 0 against the exact spectrum (SURVEY §8(c)
    "open-z, large N"): with Z4 vectors E[m_n] = tr T_n(H~) and Var(m_n) = sum_{i!=j}
    |T_n(H~)_ij|^2 <= ||T_n(H~)||_F^2 = sum_k T_n(x_k)^2, so every mu_n must lie within 6 of
    these (upper-bound) standard deviations of the exact trace; a dropped term, sign or
    scale error moves mu_n by O(N) >> sigma ~ sqrt(N/R).  mu_0 = N exactly."""
    from bloch_ref import cheb_moments, slab_energies

    lat, rp, col, val, a, b = problem((200, 100, 40), potential=ZERO_POTENTIAL)
    M, R = 200, 32
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, _ = ctx.moments(M, R, SEED, want_eta=False)
    x = a * (slab_energies(lat, rp, col, val) - b)
    assert np.max(np.abs(x)) < 1
    tr, sq = cheb_moments(x, M)
    sigma = np.sqrt(sq / R)
    z = np.abs(mu - tr) / sigma
    assert mu[0] == lat.n
    assert np.max(z[1:]) < 6.0, (np.argmax(z), np.max(z))
    assert np.sqrt(np.mean(z[1:] ** 2)) < 1.5


def test_check_hermitian_flag(pkg):
    """KPM_CHECK_HERMITIAN: the TI matrix passes (host and device CSR); a broken conjugate
    pair or a one-sided entry is rejected with KPM_EINVAL; without the flag it is accepted."""
    import torch

    lat, rp, col, val, a, b = problem((4, 5, 6))
    with pkg.KpmContext(check_hermitian=True) as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        d = [torch.from_numpy(x).cuda() for x in (rp, col, val.view(np.float64))]
        ctx.set_matrix(*d, a, b, mem=pkg.KPM_MEM_DEVICE)
        mu, _ = ctx.moments(16, 4, SEED)
        assert mu[0] == lat.n
        k = int(np.nonzero(col[rp[0]:rp[1]] != 0)[0][0])  # an off-diagonal entry of row 0
        bad = val.copy()
        bad[k] += 1e-6j
        with pytest.raises(pkg.KpmError) as e:
            ctx.set_matrix(rp, col, bad, a, b)
        assert e.value.status == pkg.KPM_EINVAL and "not Hermitian" in str(e.value)
    # row 0 gets an extra entry to column n-1 whose partner is missing
    rp2 = rp.copy()
    rp2[1:] += 1
    col2 = np.insert(col, rp[1], lat.n - 1)
    val2 = np.insert(val, rp[1], 0.25 + 0j)
    with pkg.KpmContext(check_hermitian=True) as ctx:
        with pytest.raises(pkg.KpmError) as e:
            ctx.set_matrix(rp2, col2, val2, a, b)
        assert e.value.status == pkg.KPM_EINVAL
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp2, col2, val2, a, b)  # unchecked by default


def test_c3_full_m_r16(pkg):
    """C3 at M = 2000 with the R = 16 default (the bench's by_R entry; 8-lane block-cache map,
    library order): columns 0 and 15 element by element against the oracle."""
    lat, rp, col, val, a, b = problem((200, 100, 40))
    M, R = 2000, 16
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, eta = ctx.moments(M, R, SEED)
        assert ctx.last_kernel() == pkg.variant_name(R, 0)
    assert mu[0] == lat.n
    threads = oracle.max_threads()
    for c in (0, 15):
        eta_o = oracle.kpm_eta(rp, col, val, a, b, M, 1, SEED, col_begin=c, threads=threads)
        check(eta[c : c + 1], None, eta_o, cols=[0])


def test_bench_config_c3_full_m(pkg):
    """The headline configuration exactly as bench.py times it: C3 200x100x40, M = 2000, R = 32,
    the width's default kernel and the library's default chunk order.  Columns 0, 7, 19, 31
    element by element against the oracle (1e-10 per column, R10; ~2 min of oracle
    time), bitwise run-to-run reproducible, mu_0 = N."""
    lat, rp, col, val, a, b = problem((200, 100, 40))
    M, R = 2000, 32
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        mu, eta = ctx.moments(M, R, SEED)
        assert ctx.last_kernel() == pkg.variant_name(R, 0)
        mu2, eta2 = ctx.moments(M, R, SEED)
    assert np.array_equal(eta, eta2) and np.array_equal(mu, mu2)
    assert mu[0] == lat.n and np.all(np.abs(mu) <= mu[0])
    threads = oracle.max_threads()
    for c in (0, 7, 19, 31):
        eta_o = oracle.kpm_eta(rp, col, val, a, b, M, 1, SEED, col_begin=c, threads=threads)
        check(eta[c : c + 1], None, eta_o, cols=[0])


@pytest.mark.parametrize("R", [1, 32])
def test_z4_start_block_bit_exact(pkg, R):
    """|rand()>: the device Z4 block equals the oracle's independent Philox copy bit for
    bit -- read back through the plain SpMMV W = H V with H = 1 (exact), on a ragged row count."""
    n = 1000
    rp = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int64)
    val = np.ones(n, dtype=np.complex128)
    seed = 0x5EED + R
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, 1.0, 0.0)
        _, w = ctx.sweep_kernel("spmmv", R, seed, n_sweeps=1, want_w=True)
    assert np.array_equal(w, oracle.z4_block(0, n, 0, R, seed))


def test_z4_later_column_blocks_exact_arithmetic(pkg):
    """Columns 32..63 (the second block of 32, col_begin = 32) and the per-column stage (col_begin
    = r): on a ring with hopping 1, a = 1/4, b = 0 every eta is a dyadic rational computed exactly,
    so GPU and oracle agree bit for bit iff their start vectors do."""
    n = 4000
    i = np.arange(n)
    rows = np.concatenate([i, i])
    cols = np.concatenate([(i + 1) % n, (i - 1) % n])
    order = np.lexsort((cols, rows))
    col = cols[order].astype(np.int64)
    rp = np.arange(0, 2 * n + 1, 2, dtype=np.int64)
    val = np.ones(2 * n, dtype=np.complex128)
    M, R, seed = 8, 64, 99
    eta_o = oracle.kpm_eta(rp, col, val, 0.25, 0.0, M, R, seed)
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, 0.25, 0.0)
        _, eta = ctx.moments(M, R, seed)
        _, eta1 = ctx.moments_stage("aug_spmv", M, 4, seed)
    assert np.array_equal(eta, eta_o)
    assert np.array_equal(eta1, eta_o[:4])


def test_per_sweep_timing(pkg):
    """KPM_TIMING: one device time per sweep (init + M/2 - 1 main sweeps), consistent with the
    call's total; without the flag no per-sweep times."""
    lat, rp, col, val, a, b = problem((8, 8, 8))
    with pkg.KpmContext(flags=pkg.KPM_TIMING | pkg.KPM_DETERMINISTIC) as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        ctx.moments(64, 4, SEED)
        t = ctx.sweep_times()
        total, sweep, n = ctx.last_timing()
    assert len(t) == 32 and np.all(t > 0) and t.sum() <= total * 1.001
    assert abs(np.mean(t[1:]) - sweep) <= 0.05 * sweep + 1e-3
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        ctx.moments(64, 4, SEED)
        assert len(ctx.sweep_times()) == 0


def test_fig1_demo_small(pkg, tmp_path):
    """The Fig. 1 demo (scripts/fig1_demo.py) end to end on one GPU at a small
    size: device-generated CSR, library order, Jackson DOS; mu_0 = N and the DOS integrates to N."""
    import json
    import os
    import subprocess
    import sys

    out = tmp_path / "dos.csv"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, f"{root}/scripts/fig1_demo.py", "--lattice", "40,40,40", "--M", "200",
                          "--R", "8", "--out", str(out)], capture_output=True, text=True, timeout=600, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    d = json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][-1])
    assert d["mu0"] == d["N"] == 4 * 40 * 40 * 40
    assert d["integral_rho"] == pytest.approx(d["N"], rel=1e-9)
    assert out.exists()


@pytest.mark.parametrize("R", [1, 8, 32])
def test_degenerate_sizes(pkg, R):
    """Degenerate cases of the method: a 1x1 matrix (one chunk of 31 padding rows), M = 2 (the
    init sweep only, mu = (eta_0, eta_1)), M = 4 (one main sweep, no CUDA graph), a matrix with
    empty rows and a row of only a diagonal; each against the oracle."""
    cases = []
    cases.append((np.array([0, 1]), np.array([0]), np.array([0.3 + 0j]), 0.9, 0.1))  # H = (0.3)
    n = 70  # a tridiagonal chain with rows 5 and 40 empty, row 63 a lone diagonal
    rows, cols, vals = [], [], []
    for i in range(n):
        if i in (5, 40):
            continue
        if i == 63:
            rows.append(i), cols.append(i), vals.append(0.7 + 0j)
            continue
        for j, v in ((i - 1, 0.5 - 0.25j), (i + 1, 0.5 + 0.25j)):
            if 0 <= j < n and j not in (5, 40, 63):
                rows.append(i), cols.append(j), vals.append(v)
    rows, cols, vals = np.array(rows), np.array(cols), np.array(vals, dtype=np.complex128)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    cases.append((np.cumsum(rp), cols.astype(np.int64), vals, 0.45, 0.0))
    for rp, col, val, a, b in cases:
        for M in (2, 4, 30):
            with pkg.KpmContext() as ctx:
                ctx.set_matrix(rp, col, val, a, b)
                mu, eta = ctx.moments(M, R, SEED)
            eta_o = oracle.kpm_eta(rp, col, val, a, b, M, R, SEED)
            check(eta, mu, eta_o)
            assert mu[0] == len(rp) - 1


@pytest.mark.parametrize("R", [1, 8, 32])
def test_closed_forms_without_oracle(pkg, R):
    """Pins of the CUDA path that need no oracle (mu_n = <v|T_n(H~)|v> averaged over
    unit-modulus v): a diagonal H has mu_n = sum_i T_n(a (lambda_i - b)) exactly for every Z4
    column, on a ragged multi-chunk size with the width's default kernel; an H with no stored
    entry at all (every chunk empty) is H~ = -a b 1, mu_n = N T_n(-a b)."""
    rng = np.random.default_rng(3)
    n = 50_001
    lam = rng.uniform(-4.0, 4.0, n)
    rp = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int64)
    a, b, M = 0.9 / 4.5, 0.3, 200
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(rp, col, lam.astype(np.complex128), a, b)
        mu, _ = ctx.moments(M, R, SEED)
    x = a * (lam - b)
    ref = np.array([np.cos(k * np.arccos(x)).sum() for k in range(M)])
    assert mu[0] == n
    assert np.max(np.abs(mu - ref)) / n <= TOL
    n0 = 1000
    with pkg.KpmContext() as ctx:
        ctx.set_matrix(np.zeros(n0 + 1, dtype=np.int64), np.zeros(0, dtype=np.int64), np.zeros(0, dtype=np.complex128),
                       0.5, 1.2)
        mu, _ = ctx.moments(40, R, SEED)
    ref0 = n0 * np.cos(np.arange(40) * np.arccos(-0.5 * 1.2))
    assert np.max(np.abs(mu - ref0)) / n0 <= TOL
