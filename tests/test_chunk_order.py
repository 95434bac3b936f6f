"""CPU tests of the library's default chunk order (kpm_plan_chunk_order, csrc/chunk_order.cpp;
DESIGN.md §7 "Chunk order"): derived from the matrix's chunk adjacency alone, it equals the
TI-specific walks written out in workloads.ti_lattice (y-lines, 2-line strips; lock-step rounds
of the launch grid, leftovers in balanced lock-step segments) on the paper's lattices, with and
without the multi-rank edge split, and is a permutation for any input."""
import numpy as np
import pytest

from workloads.ti_lattice import Lattice, chunk_order_ylines, chunk_order_ystrips, generate_csr

C = 32


@pytest.fixture(scope="module")
def pkg():
    from paper_1410_5242_b200 import build

    build.build()
    import paper_1410_5242_b200 as p

    return p


def block_neighbours(rp, col, n):
    """Chunk b is a block neighbour of chunk c if c's rows reference all 32 rows of b (numpy,
    independent of the library's run lists)."""
    nch = (n + C - 1) // C
    ptr, nbr = [0], []
    for c in range(nch):
        cols = np.unique(col[rp[c * C]:rp[min((c + 1) * C, n)]])
        blocks, counts = np.unique(cols // C, return_counts=True)
        full = [int(b) for b, k in zip(blocks, counts) if k == C and b != c]
        nbr += full
        ptr.append(len(nbr))
    return np.array(ptr), np.array(nbr, dtype=np.int64)


@pytest.mark.parametrize("dims,grid", [((200, 100, 40), 148), ((20, 12, 16), 148), ((30, 7, 8), 16), ((9, 40, 24), 7)])
def test_line_walk_matches_ylines_twin(pkg, dims, grid):
    lat = Lattice(*dims)
    rp, col, _ = generate_csr(lat)
    ptr, nbr = block_neighbours(rp, col, lat.n)
    got = pkg.plan_chunk_order(ptr, nbr, grid)
    assert np.array_equal(np.sort(got), np.arange(len(ptr) - 1))
    assert np.array_equal(got, chunk_order_ylines(lat, grid))


@pytest.mark.parametrize("dims,grid", [((12, 10, 16), 20), ((6, 30, 8), 9)])
def test_edges_last_matches(pkg, dims, grid):
    """Multi-rank split: the x-slab's first and last planes (edge chunks) stay out of the lines."""
    lat = Lattice(*dims)
    rp, col, _ = generate_csr(lat)
    ptr, nbr = block_neighbours(rp, col, lat.n)
    zb = 4 * lat.nz // C
    per_plane = lat.ny * zb
    nch = len(ptr) - 1
    skip = np.zeros(nch, dtype=np.int8)
    skip[:per_plane] = 1
    skip[nch - per_plane:] = 1
    got = pkg.plan_chunk_order(ptr, nbr, grid, skip=skip)
    assert np.array_equal(got, chunk_order_ylines(lat, grid, edges_last=True))


@pytest.mark.parametrize("dims,grid", [((200, 100, 40), 148), ((21, 12, 16), 10), ((8, 9, 8), 3)])
def test_strip_walk_matches_ystrips(pkg, dims, grid):
    """width 2: strips of two x-adjacent y-lines walked step by step (the R = 32 kernel's order)."""
    lat = Lattice(*dims)
    rp, col, _ = generate_csr(lat)
    ptr, nbr = block_neighbours(rp, col, lat.n)
    got = pkg.plan_chunk_order(ptr, nbr, grid, width=2)
    assert np.array_equal(got, chunk_order_ystrips(lat, grid))


def test_permutation_for_arbitrary_graphs(pkg):
    rng = np.random.default_rng(3)
    for n in (1, 5, 300):
        ptr = np.concatenate([[0], np.cumsum(rng.integers(0, 6, n))])
        nbr = rng.integers(0, n, ptr[-1])
        for grid in (1, 3, 148):
            for width in (1, 2):
                got = pkg.plan_chunk_order(ptr, nbr, grid, width=width)
                assert np.array_equal(np.sort(got), np.arange(n))
    with pytest.raises(pkg.KpmError):
        pkg.plan_chunk_order([0, 1], [5], 4)


def test_leftover_segments_balanced(pkg):
    """Lines left after the last full round are cut into `grid` contiguous, balanced segments:
    CTA b (positions b, b + G, ... after the rounds) walks consecutive chunks of one line."""
    lat = Lattice(7, 10, 8)  # 7 lines of length 10 (zb = 1): with G = 3, 2 rounds + 1 line left
    rp, col, _ = generate_csr(lat)
    ptr, nbr = block_neighbours(rp, col, lat.n)
    G = 3
    got = pkg.plan_chunk_order(ptr, nbr, G)
    rest = got[2 * 3 * 10:]  # after 2 rounds of 3 lines x 10 steps
    per_cta = [rest[b::G] for b in range(G)]
    assert sorted(len(p) for p in per_cta) == [3, 3, 4]
    for p in per_cta:  # each segment: consecutive y-steps of the leftover line (chunk offset 1)
        assert np.all(np.diff(p) == 1)
