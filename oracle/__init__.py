"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Python side of the plain CPU oracle (see kpm_oracle.cpp for the passages it follows).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this package.  The product package paper_1410_5242_b200 never imports
it and shares no code with it.

Functions whose parity is not pinned against the paper or mathematics say so here and
in DESIGN.md ("parity unpinned"): none at present -- every public function below is
pinned by a test in tests/test_oracle_pins.py or tests/test_sell_ref.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kpm_oracle.cpp")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

CHAINED = 0  # Fig. 3 BLAS-1 chain
FUSED = 1  # Fig. 4 aug_spmv per row


def build(force: bool = False) -> str:
    """Compile oracle/liboracle.so with g++ (plain -O2, no FMA contraction, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", tmp, _SRC]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64, i32, dbl, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint64
        p = ctypes.c_void_p
        lib.ora_philox4x32_10.argtypes = [p, p, p]
        lib.ora_philox4x32_10.restype = None
        lib.ora_z4_block.argtypes = [i64, i64, i64, i32, u64, p]
        lib.ora_z4_block.restype = None
        lib.ora_kpm_eta_v0.argtypes = [i64, p, p, p, dbl, dbl, i32, i32, p, i32, i32, p]
        lib.ora_kpm_eta_v0.restype = i32
        lib.ora_kpm_eta.argtypes = [i64, p, p, p, dbl, dbl, i32, i32, u64, i64, i32, i32, p]
        lib.ora_kpm_eta.restype = i32
        lib.ora_eta_to_mu.argtypes = [i32, i32, p, p, p]
        lib.ora_eta_to_mu.restype = None
        lib.ora_max_threads.argtypes = []
        lib.ora_max_threads.restype = i32
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    _load().ora_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def z4_block(row_begin: int, n_rows: int, col_begin: int, R: int, seed: int) -> np.ndarray:
    """Start block |rand()> as complex128 (n_rows, R), row-major."""
    out = np.zeros((n_rows, R), dtype=np.complex128)
    _load().ora_z4_block(row_begin, n_rows, col_begin, R, seed, _ptr(out))
    return out


def _csr(row_ptr, col, val):
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    c = np.ascontiguousarray(col, dtype=np.int64)
    v = np.ascontiguousarray(val, dtype=np.complex128)
    return rp, c, v


def kpm_eta(row_ptr, col, val, a, b, M, R, seed, col_begin=0, mode=FUSED, threads=0) -> np.ndarray:
    """eta_n^(r), complex (R, M), with Z4 Philox start vectors of global columns
    col_begin..col_begin+R-1 (Fig. 3 / Fig. 4 column by column)."""
    rp, c, v = _csr(row_ptr, col, val)
    n = len(rp) - 1
    eta = np.zeros((R, M), dtype=np.complex128)
    st = _load().ora_kpm_eta(n, _ptr(rp), _ptr(c), _ptr(v), a, b, M, R, seed, col_begin, mode,
                             threads, _ptr(eta))
    if st != 0:
        raise ValueError(f"oracle rejected arguments (status {st})")
    return eta


def kpm_eta_v0(row_ptr, col, val, a, b, M, v0, mode=FUSED, threads=0) -> np.ndarray:
    """eta for explicit start block v0 (complex (n, R))."""
    rp, c, v = _csr(row_ptr, col, val)
    n = len(rp) - 1
    v0 = np.ascontiguousarray(v0, dtype=np.complex128)
    if v0.ndim == 1:
        v0 = v0[:, None]
    assert v0.shape[0] == n
    R = v0.shape[1]
    eta = np.zeros((R, M), dtype=np.complex128)
    st = _load().ora_kpm_eta_v0(n, _ptr(rp), _ptr(c), _ptr(v), a, b, M, R, _ptr(v0), mode,
                                threads, _ptr(eta))
    if st != 0:
        raise ValueError(f"oracle rejected arguments (status {st})")
    return eta


def eta_to_mu(eta: np.ndarray):
    """(mu (M,), m (R, M) complex) from eta (R, M) by the doubling identities."""
    eta = np.ascontiguousarray(eta, dtype=np.complex128)
    R, M = eta.shape
    mu = np.zeros(M)
    m = np.zeros((R, M), dtype=np.complex128)
    _load().ora_eta_to_mu(M, R, _ptr(eta), _ptr(mu), _ptr(m))
    return mu, m


def max_threads() -> int:
    return int(_load().ora_max_threads())


# ---------------------------------------------------------------- DOS (NEXT #1) ----
def jackson(M: int) -> np.ndarray:
    """Jackson kernel g_n, n = 0..M-1 (Weisse et al., Rev. Mod. Phys. 78, 275 (2006) -- the
    KPM review the paper cites as [Weisse06]):
        g_n = [(M - n + 1) cos(pi n/(M+1)) + sin(pi n/(M+1)) cot(pi/(M+1))] / (M+1)."""
    n = np.arange(M, dtype=np.float64)
    q = np.pi / (M + 1)
    return ((M - n + 1) * np.cos(q * n) + np.sin(q * n) / np.tan(q)) / (M + 1)


def chebyshev_nodes(K: int) -> np.ndarray:
    """x_k = cos(pi (k + 1/2) / K), k = 0..K-1."""
    return np.cos(np.pi * (np.arange(K) + 0.5) / K)


def dos(mu, a, b, K=None, energies=None, kernel="jackson"):
    """Density of states rho(E) of H from mu_n = tr T_n(H~) (Eq. (2) `DOS`; the
    reconstruction step of P:258-260):
        rho~(x) = [g_0 mu_0 + 2 sum_{n>=1} g_n mu_n T_n(x)] / (pi sqrt(1 - x^2)),
        E = x/a + b,  rho(E) = a rho~(a (E - b)).
    Evaluated at `energies`, or at the K Chebyshev nodes.  Returns (E, rho)."""
    mu = np.asarray(mu, dtype=np.float64)
    M = len(mu)
    g = jackson(M) if kernel == "jackson" else np.ones(M)
    if energies is None:
        x = chebyshev_nodes(K if K else 2 * M)
    else:
        x = a * (np.asarray(energies, dtype=np.float64) - b)
    t_prev, t = np.ones_like(x), x.copy()
    s = g[0] * mu[0] * t_prev
    if M > 1:
        s = s + 2.0 * g[1] * mu[1] * t
    for n in range(2, M):  # T_n by the three-term recurrence
        t_prev, t = t, 2.0 * x * t - t_prev
        s = s + 2.0 * g[n] * mu[n] * t
    rho_x = s / (np.pi * np.sqrt(1.0 - x * x))
    return x / a + b, a * rho_x
