"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Independent numpy reference for the integer/byte work of the hot path's setup step
(SURVEY §8(a) a0): the SELL-C-sigma layout (Kreutzer et al., cited at PAPER.md P:126-128;
"CRS format (similar to SELL-1)") and the row-block halo maps of a
data-parallel row distribution.  The product library builds both
in C++ (paper_1410_5242_b200/csrc/); tests compare its exports with these bit for bit.

Layout contract:
  * local rows 0..n_loc-1; sigma-windows [w*sigma, (w+1)*sigma) are stably sorted by row
    length, descending (sigma = 1: identity).  perm[p] = local row stored at position p.
  * chunk c holds positions [c*C, (c+1)*C); clen[c] = max length of its rows (0 for
    padding positions p >= n_loc); cptr[c] = sum_{c' < c} C * clen[c'] (int64).
  * entry j of the row at position p = c*C + k lives at cptr[c] + j*C + k (column-major
    inside the chunk); within-row entry order: the row's own-position (diagonal) entry
    first, if stored (first occurrence), then the other entries in CSR order.
  * columns are renumbered: a local column i becomes invperm[i]; a column owned by
    another rank becomes n_pad + h, n_pad = n_chunks*C, h = its slot in the halo list.
  * padding slots: value 0 + 0i, column = p (the slot's own position).
Halo list: all distinct remote global columns, ordered by (owner rank, global column).
"""
from __future__ import annotations

import numpy as np


def owner_of(cols: np.ndarray, row_begins: np.ndarray) -> np.ndarray:
    """Owning rank of each global column for the row ranges [row_begins[q], row_begins[q+1])."""
    return np.searchsorted(row_begins, cols, side="right") - 1


def halo_list(col: np.ndarray, row_begin: int, row_end: int, row_begins: np.ndarray):
    """Sorted distinct remote columns (by owner, then column) and their owners."""
    remote = col[(col < row_begin) | (col >= row_end)]
    uniq = np.unique(remote)  # ascending global column == ascending (owner, column)
    return uniq, owner_of(uniq, row_begins)


def build_sell(row_ptr, col, val, C=32, sigma=1, row_begin=0, row_end=None, row_begins=None):
    """Reference SELL-C-sigma of the CSR rows [row_begin, row_end) with global columns.
    Returns dict(val complex128, col int32, cptr int64, clen int32, perm int32,
    n_pad, halo (global cols), halo_owner)."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    val = np.asarray(val, dtype=np.complex128)
    n_loc = len(row_ptr) - 1
    if row_end is None:
        row_end = row_begin + n_loc
    assert row_end - row_begin == n_loc
    if row_begins is None:
        row_begins = np.array([row_begin, row_end], dtype=np.int64)
    lens = np.diff(row_ptr)

    # sigma-window stable sort by descending length
    perm = np.arange(n_loc, dtype=np.int64)
    if sigma > 1:
        for w0 in range(0, n_loc, sigma):
            w1 = min(w0 + sigma, n_loc)
            order = np.argsort(-lens[w0:w1], kind="stable")
            perm[w0:w1] = w0 + order
    invperm = np.empty_like(perm)
    invperm[perm] = np.arange(n_loc)

    n_chunks = (n_loc + C - 1) // C
    n_pad = n_chunks * C
    lens_pos = np.zeros(n_pad, dtype=np.int64)
    lens_pos[:n_loc] = lens[perm]
    clen = lens_pos.reshape(n_chunks, C).max(axis=1)
    cptr = np.zeros(n_chunks + 1, dtype=np.int64)
    np.cumsum(C * clen, out=cptr[1:])
    total = int(cptr[-1])

    # padding defaults: value 0, column = own position
    s_val = np.zeros(total, dtype=np.complex128)
    chunk_of_slot = np.repeat(np.arange(n_chunks), C * clen)
    within = np.arange(total) - np.repeat(cptr[:-1], C * clen)
    s_col = chunk_of_slot * C + within % C

    # column renumbering
    halo, halo_owner = halo_list(col, row_begin, row_end, np.asarray(row_begins))
    local = (col >= row_begin) & (col < row_end)
    new_col = np.empty_like(col)
    new_col[local] = invperm[col[local] - row_begin]
    new_col[~local] = n_pad + np.searchsorted(halo, col[~local])

    # scatter entries: row i at position p = invperm[i], entry j -> cptr[p//C] + j*C + p%C.
    # Entry order within a row: the row's own-position (diagonal) entry first, if stored
    # (its first occurrence), then the other entries in stored order (R18).
    rows = np.repeat(np.arange(n_loc), lens)
    j = np.arange(len(col)) - np.repeat(row_ptr[:-1], lens)
    p = invperm[rows]
    is_diag = new_col == p
    jd = np.full(n_loc, np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(jd, rows[is_diag], j[is_diag])
    jd_e = jd[rows]
    has_d = jd_e != np.iinfo(np.int64).max
    j = np.where(has_d & (j == jd_e), 0, np.where(has_d & (j < jd_e), j + 1, j))
    dest = cptr[p // C] + j * C + p % C
    s_val[dest] = val
    s_col[dest] = new_col
    if n_pad + len(halo) > np.iinfo(np.int32).max:
        raise OverflowError("local rows + halo exceed int32")
    return dict(val=s_val, col=s_col.astype(np.int32), cptr=cptr, clen=clen.astype(np.int32),
                perm=perm.astype(np.int32), n_pad=n_pad, halo=halo, halo_owner=halo_owner)


def sell_to_csr_entries(s, n_loc, C=32):
    """Entry set {(local position row, column, value)} of a SELL matrix, padding dropped
    (round trip helper)."""
    out = []
    n_chunks = len(s["clen"])
    for c in range(n_chunks):
        for k in range(C):
            p = c * C + k
            if p >= n_loc:
                continue
            for jj in range(int(s["clen"][c])):
                idx = int(s["cptr"][c]) + jj * C + k
                out.append((p, int(s["col"][idx]), complex(s["val"][idx])))
    return out


def send_lists(cols_by_rank, row_begins):
    """For every (owner q, requester p): sorted global rows of q that p needs.
    cols_by_rank[p] = global columns referenced by rank p's rows."""
    P = len(row_begins) - 1
    out = {}
    for p in range(P):
        halo, owner = halo_list(np.asarray(cols_by_rank[p]), row_begins[p], row_begins[p + 1],
                                np.asarray(row_begins))
        for q in range(P):
            need = halo[owner == q]
            if len(need):
                out[(q, p)] = need
    return out
