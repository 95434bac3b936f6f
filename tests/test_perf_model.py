"""The bench's roofline arithmetic against the paper's own numbers (Eq. (9)-(10),
`eq:codebalance_topi`): with N_nzr = 13 nonzeros per row,
B_min(R) = (260/R + 48)/138 byte/flop, B_min(1) = 2.23, B_min(inf) = 0.35."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("R", [1, 2, 4, 8, 16, 32, 1024])
def test_code_balance_matches_paper(bench, R):
    n = 1000
    nnz = 13 * n
    B = bench.alg_bytes_per_sweep(n, nnz, R) / bench.alg_flops_per_sweep(n, nnz, R)
    assert B == pytest.approx((260 / R + 48) / 138, rel=1e-15)


def test_code_balance_limits(bench):
    n, nnz = 10, 130
    b1 = bench.alg_bytes_per_sweep(n, nnz, 1) / bench.alg_flops_per_sweep(n, nnz, 1)
    binf = bench.alg_bytes_per_sweep(n, nnz, 10**9) / bench.alg_flops_per_sweep(n, nnz, 10**9)
    assert round(b1, 2) == 2.23 and round(binf, 2) == 0.35


def test_c3_numbers_of_the_survey(bench):
    """C3 at R = 32: 5.74 GB and 14.05 GF per sweep (N_nz = 13N - 16NxNy)."""
    n = 200 * 100 * 40 * 4
    nnz = 13 * n - 16 * 200 * 100
    assert bench.alg_bytes_per_sweep(n, nnz, 32) == 5_740_800_000
    assert bench.alg_flops_per_sweep(n, nnz, 32) == pytest.approx(14.049e9, rel=1e-4)


def test_both_arms_emit_the_same_config(bench):
    """bench.py's reference arm and its own arm build `config` with one function (the driver's
    same_config check)."""
    import argparse

    for cfg, world in (("bar", 1), ("bar", 4), ("C4", 2)):
        args = argparse.Namespace(config=cfg, lattice="200,100,40", M=None, R=None)
        w = bench.workload(args, world)
        c = bench.config_dict(w, world)
        assert c["workload"] == w["name"] and c["parallelism"] == f"x-slab dp{world}"
        assert set(c) == {"workload", "lattice", "M", "R", "parallelism", "l2"}
        assert c["l2"].startswith("no flush: inputs larger than L2")  # C3 slabs, C4: GBs per GPU
