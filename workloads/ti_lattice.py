"""Seeded synthetic inputs shared by the CUDA path's harness and the oracle's tests.

This module builds the *input* of the KPM hot path -- the sparse Hamiltonian H of the
3D topological insulator (Eq. (1) `Ham`) and the spectral
rescaling a, b (Gershgorin) -- and nothing of the method's arithmetic
(no Chebyshev recurrence, no dot products, no moments).  Both `oracle/` and the
product path consume what it produces; neither imports the other.

Readings of the paper:
  * Gamma^0 = 1_4, Gamma^1 = tau_z (x) 1, Gamma^2 = tau_x (x) s_x,
    Gamma^3 = tau_x (x) s_y, Gamma^4 = tau_x (x) s_z   ("4x4 Dirac matrices", P:188;
    "precise form ... not relevant"); t = 1.
  * periodic x and y, open z ("Periodic boundary conditions in the x and y
    directions").
  * row = 4*(z + Nz*(y + Ny*x)) + o, orbital o = 2*tau + s fastest, x slowest, so
    the x-wrap gives the "outlying diagonals in the matrix corners" and an
    x-slab is a contiguous row block.
  * quantum-dot superlattice potential (profile not in the paper):
    V_n = V_d on the top layer z = Nz-1 where x mod S_x < D_x and y mod S_y < D_y.
  * H_{n+e_j, n} = -t (Gamma^1 - i Gamma^{j+1}) / 2,  H_{n, n+e_j} = its adjoint,
    H_{n,n} = V_n Gamma^0 + 2 Gamma^1   (Eq. (1)).

Per-row entry order (the order the CSR stores and the SELL format preserves):
neighbour sites  -x, -y, -z, on-site, +z, +y, +x ; inside a neighbour block the
entries are in ascending orbital column.  Structural zeros of the 4x4 blocks are
dropped, so bulk rows have 13 nonzeros ("N_nz ~ 13N") and z-surface rows 11.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# ---- Gamma matrices (orbital index o = 2*tau + s, Kronecker order tau (x) s) --------
_s0 = np.eye(2, dtype=np.complex128)
_sx = np.array([[0, 1], [1, 0]], dtype=np.complex128)
_sy = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
_sz = np.array([[1, 0], [0, -1]], dtype=np.complex128)

GAMMA = (
    np.eye(4, dtype=np.complex128),  # Gamma^0
    np.kron(_sz, _s0),  # Gamma^1
    np.kron(_sx, _sx),  # Gamma^2
    np.kron(_sx, _sy),  # Gamma^3
    np.kron(_sx, _sz),  # Gamma^4
)
GAMMA5 = np.kron(_sy, _s0)  # anticommutes with Gamma^1..Gamma^4 (chiral partner)

T_HOP = 1.0


def hop_block(j: int, t: float = T_HOP) -> np.ndarray:
    """H_{n+e_j, n} = -t (Gamma^1 - i Gamma^{j+1}) / 2, j in {1,2,3} (Eq. (1))."""
    return -t * (GAMMA[1] - 1j * GAMMA[j + 1]) / 2.0


def onsite_block(v: float) -> np.ndarray:
    """H_{n,n} = V_n Gamma^0 + 2 Gamma^1 (Eq. (1))."""
    return v * GAMMA[0] + 2.0 * GAMMA[1]


@dataclass(frozen=True)
class Superlattice:
    """Quantum-dot superlattice V_n; our stand-in profile."""

    spacing: tuple[int, int] = (20, 20)
    dot: tuple[int, int] = (6, 6)
    depth: float = 0.5


ZERO_POTENTIAL = Superlattice(depth=0.0)
DEFAULT_POTENTIAL = Superlattice()


@dataclass(frozen=True)
class Lattice:
    nx: int
    ny: int
    nz: int
    potential: Superlattice = DEFAULT_POTENTIAL
    periodic_z: bool = False  # tests only (Bloch closed form); the paper's samples are open in z

    @property
    def n(self) -> int:
        """Matrix dimension N = 4 Nx Ny Nz."""
        return 4 * self.nx * self.ny * self.nz

    @property
    def rows_per_plane(self) -> int:
        return 4 * self.ny * self.nz

    def nnz_expected(self) -> int:
        """13N - 16 Nx Ny for open z (Nx, Ny >= 3, Nz >= 2); 13N for periodic z (Nz >= 3)."""
        if self.periodic_z:
            return 13 * self.n
        return 13 * self.n - 16 * self.nx * self.ny

    def row_of(self, x, y, z, o=0):
        return 4 * (z + self.nz * (y + self.ny * x)) + o


def _potential_plane(lat: Lattice, x: int) -> np.ndarray:
    """V_n for all (y, z) of plane x, shape (Ny, Nz)."""
    pot = lat.potential
    v = np.zeros((lat.ny, lat.nz))
    if pot.depth != 0.0 and (x % pot.spacing[0]) < pot.dot[0]:
        ys = (np.arange(lat.ny) % pot.spacing[1]) < pot.dot[1]
        v[ys, lat.nz - 1] = pot.depth
    return v


def _block_entries(block: np.ndarray):
    """Per block row o: list of (o', value) with nonzero value, ascending o'."""
    out = []
    for o in range(4):
        out.append([(op, block[o, op]) for op in range(4) if block[o, op] != 0])
    return out


def generate_csr(lat: Lattice, x0: int = 0, x1: int | None = None):
    """CSR rows of the x-planes [x0, x1): (row_ptr int64[n_loc+1], col int64[nnz] global,
    val complex128[nnz]).  Rows are [row_of(x0,0,0), row_of(x1,0,0))."""
    if x1 is None:
        x1 = lat.nx
    if not (0 <= x0 <= x1 <= lat.nx):
        raise ValueError("bad x range")
    nx, ny, nz = lat.nx, lat.ny, lat.nz
    # neighbour order: -x, -y, -z, onsite, +z, +y, +x
    # row at site s reads site s - e_j through H_{s, s-e_j} = hop_block(j)
    # and site s + e_j through H_{s, s+e_j} = hop_block(j)^dagger
    hops = {j: _block_entries(hop_block(j)) for j in (1, 2, 3)}
    hops_dag = {j: _block_entries(hop_block(j).conj().T) for j in (1, 2, 3)}
    plane_rows = lat.rows_per_plane
    n_loc = (x1 - x0) * plane_rows

    # row lengths: 13 everywhere, minus 2 for each missing z-neighbour
    z = np.arange(nz)
    site_len = np.full(nz, 13, dtype=np.int64)
    if not lat.periodic_z:
        site_len -= 2 * (z == 0) + 2 * (z == nz - 1)
    plane_len = np.repeat(np.tile(site_len, ny), 4)  # (ny*nz*4,) in row order
    lens = np.tile(plane_len, x1 - x0)
    row_ptr = np.zeros(n_loc + 1, dtype=np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz, dtype=np.complex128)

    # slot layout per row: 13 slots (2 per neighbour, 1 on-site); invalid slots masked
    Y, Z, O = np.meshgrid(np.arange(ny), np.arange(nz), np.arange(4), indexing="ij")
    Y, Z, O = Y.ravel(), Z.ravel(), O.ravel()  # row order within a plane
    nslot = 13
    base_mask = np.ones((plane_rows, nslot), dtype=bool)
    if not lat.periodic_z:
        base_mask[Z == 0, 4:6] = False  # -z slots
        base_mask[Z == nz - 1, 7:9] = False  # +z slots

    def nb_slots(entries, dest_site_row):
        """entries per orbital -> (cols (rows,2), vals (rows,2))."""
        c = np.empty((plane_rows, 2), dtype=np.int64)
        v = np.empty((plane_rows, 2), dtype=np.complex128)
        for o in range(4):
            sel = O == o
            (o_a, v_a), (o_b, v_b) = entries[o]
            c[sel, 0] = dest_site_row[sel] + o_a
            c[sel, 1] = dest_site_row[sel] + o_b
            v[sel, 0] = v_a
            v[sel, 1] = v_b
        return c, v

    pos = 0
    for x in range(x0, x1):
        xm, xp = (x - 1) % nx, (x + 1) % nx
        ym, yp = (Y - 1) % ny, (Y + 1) % ny
        zm, zp = (Z - 1) % nz, (Z + 1) % nz
        site = lambda xx, yy, zz: 4 * (zz + nz * (yy + ny * xx))  # noqa: E731
        cols = np.empty((plane_rows, nslot), dtype=np.int64)
        vals = np.empty((plane_rows, nslot), dtype=np.complex128)
        blocks = [
            (hops[1], site(xm, Y, Z)),
            (hops[2], site(x, ym, Z)),
            (hops[3], site(x, Y, zm)),
        ]
        for k, (ent, dst) in enumerate(blocks):
            cols[:, 2 * k : 2 * k + 2], vals[:, 2 * k : 2 * k + 2] = nb_slots(ent, dst)
        vpl = _potential_plane(lat, x)[Y, Z]
        own = site(x, Y, Z)
        cols[:, 6] = own + O
        vals[:, 6] = vpl + 2.0 * GAMMA[1][O, O].real
        blocks = [
            (hops_dag[3], site(x, Y, zp)),
            (hops_dag[2], site(x, yp, Z)),
            (hops_dag[1], site(xp, Y, Z)),
        ]
        for k, (ent, dst) in enumerate(blocks):
            s = 7 + 2 * k
            cols[:, s : s + 2], vals[:, s : s + 2] = nb_slots(ent, dst)
        m = base_mask
        cnt = int(m.sum())
        col[pos : pos + cnt] = cols[m]
        val[pos : pos + cnt] = vals[m]
        pos += cnt
    assert pos == nnz
    return row_ptr, col, val


def generate_csr_torch(lat: Lattice, x0: int = 0, x1: int | None = None, device="cpu", batch: int = 64):
    """The same CSR as generate_csr (identical entry order and values), built with torch on
    `device` -- for slabs too large to stage through host memory (C5: 1.5e9 nonzeros per GPU).
    Every x-plane repeats the plane template of x = 1 (neighbour planes 0, 1, 2), shifted by x
    with periodic wrap; only the diagonal potential depends on x."""
    import torch

    if x1 is None:
        x1 = lat.nx
    if lat.nx < 3:
        raise ValueError("generate_csr_torch needs Nx >= 3")
    P = lat.rows_per_plane
    zero = Lattice(lat.nx, lat.ny, lat.nz, potential=ZERO_POTENTIAL, periodic_z=lat.periodic_z)
    rp1, col1, val1 = generate_csr(zero, 1, 2)
    dx = col1 // P - 1  # -1, 0, +1
    rloc = col1 % P
    rows1 = np.repeat(np.arange(P), np.diff(rp1))
    diag = np.nonzero((dx == 0) & (rloc == rows1))[0]
    # potential of the plane's diagonal slots as a function of x (x mod S_x < D_x or not)
    pot = lat.potential
    y_of = (rows1[diag] // 4) // lat.nz
    z_of = (rows1[diag] // 4) % lat.nz
    vdot = np.where(((y_of % pot.spacing[1]) < pot.dot[1]) & (z_of == lat.nz - 1), pot.depth, 0.0)
    t = lambda a, dt=None: torch.as_tensor(a, device=device, dtype=dt)  # noqa: E731
    dx_t, rloc_t, val_t = t(dx), t(rloc), t(val1)
    diag_t, vdot_t = t(diag), t(vdot, torch.float64)
    nnz_p = len(col1)
    nplanes = x1 - x0
    row_ptr = torch.empty(nplanes * P + 1, dtype=torch.int64, device=device)
    row_ptr[0] = 0
    lens = t(np.diff(rp1)).repeat(nplanes)
    torch.cumsum(lens, 0, out=row_ptr[1:])
    col = torch.empty(nplanes * nnz_p, dtype=torch.int64, device=device)
    val = torch.empty(nplanes * nnz_p, dtype=torch.complex128, device=device)
    for b0 in range(0, nplanes, batch):
        xs = torch.arange(x0 + b0, min(x0 + b0 + batch, x1), device=device, dtype=torch.int64)
        c = ((xs[:, None] + dx_t[None, :]) % lat.nx) * P + rloc_t[None, :]
        v = val_t.repeat(len(xs), 1)
        if pot.depth != 0.0:
            on = ((xs % pot.spacing[0]) < pot.dot[0]).to(torch.float64)
            v[:, diag_t] += on[:, None] * vdot_t[None, :]
        col[b0 * nnz_p : (b0 + len(xs)) * nnz_p] = c.reshape(-1)
        val[b0 * nnz_p : (b0 + len(xs)) * nnz_p] = v.reshape(-1)
    return row_ptr, col, val


def gershgorin(row_ptr, col, val, row_begin: int = 0):
    """(lo, hi) of the union of Gershgorin discs of the given CSR rows."""
    n_loc = len(row_ptr) - 1
    rows = np.repeat(np.arange(n_loc, dtype=np.int64) + row_begin, np.diff(row_ptr))
    diag = rows == col
    absval = np.abs(val)
    radius = np.bincount(rows[~diag] - row_begin, weights=absval[~diag], minlength=n_loc)
    center = np.zeros(n_loc)
    np.add.at(center, rows[diag] - row_begin, val[diag].real)
    return float(np.min(center - radius)), float(np.max(center + radius))


def scale_factors(lo: float, hi: float, eps: float = 0.01):
    """a, b with a(H - b) mapping [lo, hi] into [-1+eps, 1-eps] (eps SPEC S:68)."""
    half = 0.5 * (hi - lo)
    b = 0.5 * (hi + lo)
    if half == 0.0:
        return 1.0 - eps, b
    return (1.0 - eps) / half, b


def dense(lat: Lattice) -> np.ndarray:
    """Dense H (tests; small lattices only)."""
    row_ptr, col, val = generate_csr(lat)
    n = lat.n
    h = np.zeros((n, n), dtype=np.complex128)
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    np.add.at(h, (rows, col), val)
    return h


def bloch_energies(lat: Lattice) -> np.ndarray:
    """Closed-form spectrum for V=0, fully periodic lattice (t=1):
    E = +-sqrt((2 - sum_j cos k_j)^2 + sum_j sin^2 k_j), each twice."""
    ks = [2 * np.pi * np.arange(n) / n for n in (lat.nx, lat.ny, lat.nz)]
    kx, ky, kz = np.meshgrid(*ks, indexing="ij")
    m = 2.0 - np.cos(kx) - np.cos(ky) - np.cos(kz)
    e = np.sqrt(m**2 + np.sin(kx) ** 2 + np.sin(ky) ** 2 + np.sin(kz) ** 2).ravel()
    return np.concatenate([e, e, -e, -e])


def chunk_order_yband(lat: Lattice, x0: int, x1: int, band: int, C: int = 32):
    """Locality hint for kpm_set_chunk_order (not method arithmetic): the SELL chunks of the
    x-slab [x0, x1) (C = 32 rows = 8 sites along z, sigma = 1, Nz % 8 == 0) ordered by y-band,
    then x, then y, then z-block, so the x-neighbour window a sweep keeps in L2 shrinks from
    2 x-planes to 2 band-planes."""
    if (4 * lat.nz) % C:
        raise ValueError("needs 8 | Nz so chunks align with z-columns")
    zb = 4 * lat.nz // C
    order = []
    for y0 in range(0, lat.ny, band):
        ys = np.arange(y0, min(y0 + band, lat.ny))
        for x in range(x1 - x0):
            base = (x * lat.ny + ys)[:, None] * zb + np.arange(zb)[None, :]
            order.append(base.ravel())
    return np.concatenate(order).astype(np.int64)


def _lockstep_segments(rest: np.ndarray, grid: int) -> np.ndarray:
    """The chunks left after the full rounds, cut into `grid` balanced contiguous segments (CTA b
    gets rest[start_b : start_b + len_b]) and laid out so that list position k*grid + b is step k
    of CTA b (the library's rule, csrc/chunk_order.cpp)."""
    n = len(rest)
    K, rem = divmod(n, grid)
    out = np.empty(n, dtype=np.int64)
    for b in range(grid):
        start, ln = b * K + min(b, rem), K + (1 if b < rem else 0)
        out[np.arange(ln) * grid + b] = rest[start:start + ln]
    return out


def chunk_order_ylines(lat: Lattice, grid: int, C: int = 32, x0: int = 0, x1: int = None, edges_last: bool = False):
    """Locality hint for kpm_set_chunk_order and the block-cache feed (not method arithmetic):
    list position b + grid*k is CTA b's k-th tile.  In full rounds of `grid` lines, CTA b
    walks one y-line of chunks (x, 0..Ny-1, z-block), all CTAs in step at the same y, so
    consecutive tiles of a CTA share their y-neighbour blocks and the x-neighbour blocks are
    other CTAs' current own blocks (L2 hits).  The lines left over after the last full round are
    cut into `grid` balanced contiguous segments walked in lock step.  Chunk ids are local to the x-slab
    [x0, x1); with edges_last (several ranks) the slab's first and last x-planes -- the edge
    chunks, launched separately -- go to the end, so the interior list keeps the rounds."""
    if (4 * lat.nz) % C:
        raise ValueError("needs 8 | Nz so chunks align with z-columns")
    zb = 4 * lat.nz // C
    nxl = (lat.nx if x1 is None else x1) - x0
    xs = np.arange(1, nxl - 1) if edges_last and nxl > 2 else np.arange(nxl)
    lines = (xs[:, None] * zb + np.arange(zb)[None, :]).ravel()  # line id = x * zb + z
    rounds = len(lines) // grid
    parts = []
    y = np.arange(lat.ny)
    for r in range(rounds):
        line = lines[r * grid:(r + 1) * grid]
        x, z = line // zb, line % zb
        parts.append(((x[None, :] * lat.ny + y[:, None]) * zb + z[None, :]).ravel())
    rest = lines[rounds * grid:]
    if len(rest):
        x, z = rest // zb, rest % zb
        parts.append(_lockstep_segments(((x[:, None] * lat.ny + y[None, :]) * zb + z[:, None]).ravel(), grid))
    if edges_last and nxl > 2:
        ex = np.array([0, nxl - 1])
        parts.append(np.sort(((ex[:, None, None] * lat.ny + y[None, :, None]) * zb
                              + np.arange(zb)[None, None, :]).ravel()))
    return np.concatenate(parts).astype(np.int64)


def chunk_order_ystrips(lat: Lattice, grid: int, C: int = 32, x0: int = 0, x1: int = None, width: int = 2):
    """Locality hint (not method arithmetic): like chunk_order_ylines, but each CTA walks a strip
    of `width` x-adjacent y-lines step by step -- tiles (x, y), (x+1, y), (x, y+1), (x+1, y+1), ...
    for width 2 -- so that, besides the y-neighbours, every tile's x-neighbour on the strip's inside
    is a block the CTA already holds.  Strips of lines (x..x+width-1, z) for x = 0, width, ...;
    rounds of `grid` strips in lock step; the leftover strips, then lines in no strip, in `grid`
    balanced lock-step segments.  The library's own order (kpm_plan_chunk_order, width 2)
    equals the width-2 form."""
    if (4 * lat.nz) % C:
        raise ValueError("needs 8 | Nz so chunks align with z-columns")
    zb = 4 * lat.nz // C
    nxl = (lat.nx if x1 is None else x1) - x0
    strips = [(x, z) for x in range(0, nxl - width + 1, width) for z in range(zb)]
    rounds = len(strips) // grid
    parts, used = [], np.zeros(nxl * lat.ny * zb, dtype=bool)
    for r in range(rounds):
        st = strips[r * grid:(r + 1) * grid]
        xs = np.array([x for x, _ in st])
        zs = np.array([z for _, z in st])
        for y in range(lat.ny):
            for dx in range(width):
                ids = ((xs + dx) * lat.ny + y) * zb + zs
                parts.append(ids)
                used[ids] = True
    rest = []
    for x, z in strips[rounds * grid:]:  # leftover strips, each walked step by step
        ids = ((x + np.arange(width)[None, :]) * lat.ny + np.arange(lat.ny)[:, None]) * zb + z
        rest.append(ids.ravel())
        used[ids.ravel()] = True
    rest.append(np.nonzero(~used)[0])
    parts.append(_lockstep_segments(np.concatenate(rest).astype(np.int64), grid))
    return np.concatenate(parts).astype(np.int64)


# ---- configurations of BASELINE.json ----------------------------------
CONFIGS = {
    "C1": dict(lattice=(8, 8, 8), M=64, R=4),
    "C2": dict(lattice=(64, 64, 32), M=1000, R=8),
    "C3": dict(lattice=(200, 100, 40), M=2000, R=32),
    "C4": dict(lattice=(400, 400, 40), M=2000, R=32),
}
SEED = 0x14105242
