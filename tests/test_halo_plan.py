"""Multi-rank index logic on the CPU: the library's halo-exchange planning (kpm_plan_recv /
kpm_plan_send, the code kpm_set_matrix runs) against the independent numpy reference
(oracle/sell_ref.py), single-process for P in {2,3,4,8} and as a real 2-process exchange
over torch.distributed gloo (the transport the library uses on the GPU is NCCL)."""
import os
import socket

import numpy as np
import pytest

from oracle import sell_ref
from workloads.ti_lattice import Lattice, generate_csr


@pytest.fixture(scope="module")
def pkg():
    from paper_1410_5242_b200 import build

    build.build()
    import paper_1410_5242_b200 as p

    return p


def slabs(lat, P):
    planes = [lat.nx * q // P for q in range(P + 1)]
    row_begins = np.array([pl * lat.rows_per_plane for pl in planes], dtype=np.int64)
    return planes, row_begins


def simulate(pkg, lat, P):
    """Every rank plans its receive runs, 'sends' its requests to the owners, owners plan
    send runs; then the data movement is simulated with global row ids as payload."""
    planes, rb = slabs(lat, P)
    recv, cols = [], []
    for p in range(P):
        rp, col, _ = generate_csr(lat, planes[p], planes[p + 1])
        cols.append(col)
        recv.append(pkg.plan_recv(rb, p, rp, col))
    sends = {}
    for q in range(P):
        for p in range(P):
            req = recv[p][recv[p][:, 0] == q][:, 1:3]
            if len(req):
                sends[(q, p)] = pkg.plan_send(rb[q], rb[q + 1], p, req)
    for p in range(P):
        halo, owner = sell_ref.halo_list(cols[p], rb[p], rb[p + 1], rb)
        got = np.full(len(halo), -1, dtype=np.int64)
        for q in range(P):
            rr = recv[p][recv[p][:, 0] == q]
            if not len(rr):
                continue
            sr = sends[(q, p)]
            assert len(sr) == len(rr)  # matched in order, run by run
            for (peer, pos, cnt), (_, g0, cnt2, slot) in zip(sr, rr):
                assert cnt == cnt2
                got[slot : slot + cnt] = rb[q] + pos + np.arange(cnt)  # sigma = 1: payload = global ids
        assert np.array_equal(got, halo)  # every halo slot holds the right global row
    return recv, sends


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_plan_matches_reference(pkg, P):
    lat = Lattice(16, 5, 8)
    recv, sends = simulate(pkg, lat, P)
    _, rb = slabs(lat, P)
    ref = sell_ref.send_lists([generate_csr(lat, *[lat.nx * q // P for q in (p, p + 1)])[1] for p in range(P)], rb)
    for (q, p), sr in sends.items():
        rows = np.concatenate([rb[q] + pos + np.arange(cnt) for _, pos, cnt in sr])
        assert np.array_equal(rows, ref[(q, p)])
    # x-slab property: one contiguous plane per neighbour and side (P >= 3), 2 runs at P = 2
    for p in range(P):
        assert len(recv[p]) == 2
        assert np.all(recv[p][:, 2] == lat.rows_per_plane)


def test_plan_rejects_foreign_request(pkg):
    with pytest.raises(pkg.KpmError):
        pkg.plan_send(100, 200, 1, [[90, 20]])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1410_5242_b200 as pkg

        lat = Lattice(12, 4, 8)
        planes, rb = slabs(lat, world)
        rp, col, _ = generate_csr(lat, planes[rank], planes[rank + 1])
        recv = pkg.plan_recv(rb, rank, rp, col)
        # requests to each owner, exchanged for real over gloo
        reqs = [recv[recv[:, 0] == o][:, 1:3].copy() for o in range(world)]
        inbox = [None] * world
        dist.all_gather_object(inbox, reqs)
        my_sends = {p: pkg.plan_send(rb[rank], rb[rank + 1], p, inbox[p][rank]) for p in range(world)
                    if len(inbox[p][rank])}
        # payload: global row ids of the sent positions
        payload = {p: np.concatenate([rb[rank] + pos + np.arange(c) for _, pos, c in sr]) for p, sr in my_sends.items()}
        box = [None] * world
        dist.all_gather_object(box, payload)
        halo, owner = sell_ref.halo_list(col, rb[rank], rb[rank + 1], rb)
        got = np.full(len(halo), -1, dtype=np.int64)
        for o in range(world):
            rr = recv[recv[:, 0] == o]
            if len(rr):
                data = box[o][rank]
                off = 0
                for _, g0, cnt, slot in rr:
                    got[slot : slot + cnt] = data[off : off + cnt]
                    off += cnt
        q.put((rank, bool(np.array_equal(got, halo)), int(len(halo))))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks(pkg):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _, _ in res) == [0, 1]
    assert all(ok for _, ok, _ in res)
    assert all(n == 2 * 4 * 4 * 8 for _, _, n in res)  # two x-planes (4*Ny*Nz rows each) per rank
