"""B200-native KPM-DOS hot path (arXiv:1410.5242): thin Python binding of libkpm.so.

Argument marshalling only -- every step of the path runs in the library's sm_100a kernels
(include/kpm.h documents the ABI).  There is no CPU fallback: importing the binding
without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libkpm.so")

KPM_OK, KPM_EINVAL, KPM_ESTATE, KPM_ERANGE, KPM_ENOMEM, KPM_ECUDA, KPM_ENCCL, KPM_EZERONORM, KPM_WDIVERGED = range(9)
KPM_MEM_HOST, KPM_MEM_DEVICE = 0, 1
KPM_CHECK_HERMITIAN, KPM_DETERMINISTIC, KPM_TIMING, KPM_VIRTUAL_RANKS = 1, 2, 4, 8
STATUS_NAMES = ["KPM_OK", "KPM_EINVAL", "KPM_ESTATE", "KPM_ERANGE", "KPM_ENOMEM", "KPM_ECUDA", "KPM_ENCCL",
                "KPM_EZERONORM", "KPM_WDIVERGED"]

# exported symbols declared in include/kpm.h
ABI_SYMBOLS = ["kpm_create", "kpm_destroy", "kpm_dos", "kpm_export_halo", "kpm_export_sell", "kpm_get_sell_info", "kpm_get_unique_id",
               "kpm_last_error", "kpm_last_kernel", "kpm_last_sweep_times", "kpm_last_timing", "kpm_moments", "kpm_moments_stage", "kpm_moments_v0",
               "kpm_plan_chunk_order", "kpm_plan_recv", "kpm_plan_send", "kpm_set_chunk_order", "kpm_set_matrix", "kpm_sweep_kernel", "kpm_variant_name", "kpm_vgroup_create",
               "kpm_vgroup_destroy"]


class KpmError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


class kpm_options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("nranks", ctypes.c_int), ("rank", ctypes.c_int),
                ("nccl_unique_id", ctypes.c_void_p), ("cuda_stream", ctypes.c_void_p), ("sell_C", ctypes.c_int),
                ("sell_sigma", ctypes.c_int), ("flags", ctypes.c_uint)]


class kpm_csr(ctypes.Structure):
    _fields_ = [("n_global", ctypes.c_int64), ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col", ctypes.c_void_p), ("val", ctypes.c_void_p),
                ("mem", ctypes.c_int)]


class kpm_sell_info(ctypes.Structure):
    _fields_ = [("n_loc", ctypes.c_int64), ("n_pad", ctypes.c_int64), ("n_chunks", ctypes.c_int64),
                ("n_slots", ctypes.c_int64), ("n_halo", ctypes.c_int64), ("C", ctypes.c_int),
                ("sigma", ctypes.c_int)]


_lib = None


def load_library():
    """Load the in-tree libkpm.so (raises if it is missing: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    P, i32, i64, u64, dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    lib.kpm_create.argtypes = [ctypes.POINTER(P), ctypes.POINTER(kpm_options)]
    lib.kpm_set_matrix.argtypes = [P, ctypes.POINTER(kpm_csr), dbl, dbl]
    lib.kpm_moments.argtypes = [P, i32, i32, u64, P, P]
    lib.kpm_moments_v0.argtypes = [P, i32, i32, P, P, P]
    lib.kpm_moments_stage.argtypes = [P, i32, i32, i32, u64, P, P]
    lib.kpm_sweep_kernel.argtypes = [P, i32, i32, u64, i32, P, P]
    lib.kpm_last_timing.argtypes = [P, P, P, P]
    lib.kpm_get_sell_info.argtypes = [P, ctypes.POINTER(kpm_sell_info)]
    lib.kpm_export_sell.argtypes = [P, P, P, P, P, P]
    lib.kpm_export_halo.argtypes = [P, P, P, P, P]
    lib.kpm_last_sweep_times.argtypes = [P, P, P]
    lib.kpm_vgroup_create.argtypes = [i32, ctypes.POINTER(P)]
    lib.kpm_vgroup_destroy.argtypes = [P]
    lib.kpm_vgroup_destroy.restype = None
    lib.kpm_last_error.argtypes = [P]
    lib.kpm_last_error.restype = ctypes.c_char_p
    lib.kpm_last_kernel.argtypes = [P]
    lib.kpm_last_kernel.restype = ctypes.c_char_p
    lib.kpm_variant_name.argtypes = [i32, i32]
    lib.kpm_variant_name.restype = ctypes.c_char_p
    lib.kpm_get_unique_id.argtypes = [P]
    lib.kpm_set_chunk_order.argtypes = [P, P, i64]
    lib.kpm_dos.argtypes = [i32, P, dbl, dbl, i32, P, i32, P, P]
    lib.kpm_plan_recv.argtypes = [i32, P, i32, P, P, P, P]
    lib.kpm_plan_send.argtypes = [i64, i64, i32, i64, P, P, P]
    lib.kpm_plan_chunk_order.argtypes = [i64, P, P, i64, i32, P, P]
    lib.kpm_destroy.argtypes = [P]
    lib.kpm_destroy.restype = None
    for name in ABI_SYMBOLS:
        if name not in ("kpm_last_error", "kpm_last_kernel", "kpm_destroy", "kpm_variant_name", "kpm_vgroup_destroy"):
            getattr(lib, name).restype = i32
    _lib = lib
    return lib


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(int(a.data_ptr()))  # torch tensor (device memory plumbing)


def variant_name(R, variant):
    """kpm_variant_name: name of kernel variant `variant` (KPM_VARIANT index) of width R, or None."""
    n = load_library().kpm_variant_name(int(R), int(variant))
    return n.decode() if n else None


def get_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0), to broadcast to the other ranks."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    st = lib.kpm_get_unique_id(buf)
    if st != KPM_OK:
        raise KpmError(st, "ncclGetUniqueId failed")
    return buf.raw


KPM_KERNEL_NONE, KPM_KERNEL_JACKSON = 0, 1


def dos(mu, a, b, K=None, energies=None, kernel="jackson"):
    """kpm_dos: (E, rho) from the moments (Jackson kernel by default)."""
    lib = load_library()
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    if energies is not None:
        energies = np.ascontiguousarray(energies, dtype=np.float64)
        K = len(energies)
    K = K or 2 * len(mu)
    E = np.zeros(K)
    rho = np.zeros(K)
    kern = KPM_KERNEL_JACKSON if kernel == "jackson" else KPM_KERNEL_NONE
    st = lib.kpm_dos(len(mu), _ptr(mu), float(a), float(b), K, _ptr(energies), kern, _ptr(E), _ptr(rho))
    if st != KPM_OK:
        raise KpmError(st, "kpm_dos")
    return E, rho


def plan_recv(row_begins, rank, row_ptr, col):
    """Receive runs (owner, first global row, count, first halo slot) -- host only."""
    lib = load_library()
    rb = np.ascontiguousarray(row_begins, dtype=np.int64)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    c = np.ascontiguousarray(col, dtype=np.int64)
    n = ctypes.c_int64(0)
    st = lib.kpm_plan_recv(len(rb) - 1, _ptr(rb), rank, _ptr(rp), _ptr(c), ctypes.byref(n), None)
    if st != KPM_OK:
        raise KpmError(st, "kpm_plan_recv")
    out = np.zeros((n.value, 4), dtype=np.int64)
    st = lib.kpm_plan_recv(len(rb) - 1, _ptr(rb), rank, _ptr(rp), _ptr(c), ctypes.byref(n), _ptr(out))
    if st != KPM_OK:
        raise KpmError(st, "kpm_plan_recv")
    return out


def plan_send(row_begin, row_end, peer, req):
    """Send runs (peer, first local position, count) answering `req` ((first, count) pairs)."""
    lib = load_library()
    rq = np.ascontiguousarray(req, dtype=np.int64).reshape(-1, 2)
    n = ctypes.c_int64(len(rq))
    out = np.zeros((max(len(rq), 1), 3), dtype=np.int64)
    st = lib.kpm_plan_send(row_begin, row_end, peer, len(rq), _ptr(rq), ctypes.byref(n), _ptr(out))
    if st != KPM_OK:
        raise KpmError(st, "kpm_plan_send")
    return out[: n.value]


def plan_chunk_order(nbr_ptr, nbr, grid, skip=None, width=1):
    """kpm_plan_chunk_order: the library's default chunk order from block-neighbour lists."""
    lib = load_library()
    nbr_ptr = np.ascontiguousarray(nbr_ptr, dtype=np.int64)
    nbr = np.ascontiguousarray(nbr, dtype=np.int64)
    n = len(nbr_ptr) - 1
    sk = None if skip is None else np.ascontiguousarray(skip, dtype=np.int8)
    out = np.zeros(max(n, 1), dtype=np.int64)
    st = lib.kpm_plan_chunk_order(n, _ptr(nbr_ptr), _ptr(nbr) if len(nbr) else None, int(grid), int(width), _ptr(sk),
                                  _ptr(out))
    if st != KPM_OK:
        raise KpmError(st, "kpm_plan_chunk_order")
    return out[:n]


class VirtualGroup:
    """kpm_vgroup_create: an in-process group of nranks virtual ranks on one device (test harness,
    KPM_VIRTUAL_RANKS in kpm.h).  Pass it as KpmContext(vgroup=...) from one thread per rank."""

    def __init__(self, nranks):
        self.lib = load_library()
        h = ctypes.c_void_p()
        st = self.lib.kpm_vgroup_create(int(nranks), ctypes.byref(h))
        if st != KPM_OK:
            raise KpmError(st, "kpm_vgroup_create")
        self.h, self.nranks = h, nranks

    def close(self):
        if getattr(self, "h", None):
            self.lib.kpm_vgroup_destroy(self.h)
            self.h = None


class KpmContext:
    """One rank's context (kpm_create ... kpm_destroy)."""

    def __init__(self, device=0, nranks=1, rank=0, nccl_unique_id=None, cuda_stream=None, sell_C=32, sell_sigma=1,
                 check_hermitian=False, flags=0, vgroup=None):
        self.lib = load_library()
        self._uid = None if nccl_unique_id is None else ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
        uid = ctypes.cast(self._uid, ctypes.c_void_p) if self._uid else None
        flags |= KPM_CHECK_HERMITIAN if check_hermitian else 0
        if vgroup is not None:
            uid, flags = vgroup.h, flags | KPM_VIRTUAL_RANKS
        opt = kpm_options(device, nranks, rank, uid, cuda_stream, sell_C, sell_sigma, flags)
        h = ctypes.c_void_p()
        st = self.lib.kpm_create(ctypes.byref(h), ctypes.byref(opt))
        if st != KPM_OK:
            raise KpmError(st, self.lib.kpm_last_error(None).decode())
        self.h = h
        self.last_status = KPM_OK

    def _check(self, st, allow=()):
        self.last_status = st
        if st != KPM_OK and st not in allow:
            raise KpmError(st, self.lib.kpm_last_error(self.h).decode())
        return st

    def set_matrix(self, row_ptr, col, val, a, b, n_global=None, row_begin=0, mem=KPM_MEM_HOST):
        """kpm_set_matrix from numpy (host) or torch (device) CSR arrays; val complex128 or
        interleaved float64."""
        keep = []
        if mem == KPM_MEM_HOST:
            row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
            col = np.ascontiguousarray(col, dtype=np.int64)
            val = np.ascontiguousarray(val)
            if val.dtype != np.complex128:
                val = np.ascontiguousarray(val, dtype=np.float64)
            keep = [row_ptr, col, val]
        n_loc = len(row_ptr) - 1
        if n_global is None:
            n_global = row_begin + n_loc
        csr = kpm_csr(n_global, row_begin, row_begin + n_loc, _ptr(row_ptr), _ptr(col), _ptr(val), mem)
        self._check(self.lib.kpm_set_matrix(self.h, ctypes.byref(csr), float(a), float(b)))
        del keep

    def set_chunk_order(self, order=None):
        """kpm_set_chunk_order: locality hint (permutation of the SELL chunks) or None."""
        if order is None:
            self._check(self.lib.kpm_set_chunk_order(self.h, None, 0))
            return
        o = np.ascontiguousarray(order, dtype=np.int64)
        self._check(self.lib.kpm_set_chunk_order(self.h, _ptr(o), len(o)))

    def moments(self, M, R, seed, want_eta=True, allow_warning=True):
        """(mu (M,), eta (R, M) complex or None)."""
        mu = np.zeros(M)
        eta = np.zeros((R, M), dtype=np.complex128) if want_eta else None
        allow = (KPM_WDIVERGED,) if allow_warning else ()
        self._check(self.lib.kpm_moments(self.h, M, R, seed, _ptr(mu), _ptr(eta)), allow)
        return mu, eta

    def moments_stage(self, stage, M, R, seed, want_eta=True):
        """kpm_moments_stage: 'naive' (Fig. 3), 'aug_spmv' (Fig. 4) or 'aug_spmmv' (Fig. 5)."""
        code = {"naive": 0, "aug_spmv": 1, "aug_spmmv": 2}[stage]
        mu = np.zeros(M)
        eta = np.zeros((R, M), dtype=np.complex128) if want_eta else None
        self._check(self.lib.kpm_moments_stage(self.h, code, M, R, seed, _ptr(mu), _ptr(eta)), (KPM_WDIVERGED,))
        return mu, eta

    def sweep_kernel(self, kind, R, seed, n_sweeps=1, want_w=False):
        """kpm_sweep_kernel: time n_sweeps of 'aug', 'aug_nodot' or 'spmmv' (the paper's Fig. 9
        kernels) at block width R; returns (ms per sweep, W (n_loc, R) complex or None)."""
        code = {"aug": 0, "aug_nodot": 1, "spmmv": 2}[kind]
        ms = ctypes.c_double(0.0)
        w = np.zeros((self.sell_info().n_loc, R), dtype=np.complex128) if want_w else None
        self._check(self.lib.kpm_sweep_kernel(self.h, code, R, seed, n_sweeps, ctypes.byref(ms), _ptr(w)))
        return ms.value, w

    def moments_v0(self, M, v0, allow=(KPM_WDIVERGED,)):
        v0 = np.ascontiguousarray(v0, dtype=np.complex128)
        if v0.ndim == 1:
            v0 = v0[:, None]
        R = v0.shape[1]
        mu = np.zeros(M)
        eta = np.zeros((R, M), dtype=np.complex128)
        self._check(self.lib.kpm_moments_v0(self.h, M, R, _ptr(v0), _ptr(mu), _ptr(eta)), allow)
        return mu, eta

    def last_timing(self):
        t, s, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        self._check(self.lib.kpm_last_timing(self.h, ctypes.byref(t), ctypes.byref(s), ctypes.byref(n)))
        return t.value, s.value, n.value

    def sweep_times(self):
        """kpm_last_sweep_times (KPM_TIMING contexts): per-sweep device ms of the last call."""
        n = ctypes.c_int64(0)
        self._check(self.lib.kpm_last_sweep_times(self.h, None, ctypes.byref(n)))
        out = np.zeros(max(n.value, 1))
        self._check(self.lib.kpm_last_sweep_times(self.h, _ptr(out), ctypes.byref(n)))
        return out[: n.value]

    def export_halo(self):
        """kpm_export_halo: (recv runs (n, 4), send runs (n, 4)) of this rank's exchange plan."""
        nr, ns = ctypes.c_int64(0), ctypes.c_int64(0)
        self._check(self.lib.kpm_export_halo(self.h, ctypes.byref(nr), None, ctypes.byref(ns), None))
        recv = np.zeros((max(nr.value, 1), 4), dtype=np.int64)
        send = np.zeros((max(ns.value, 1), 4), dtype=np.int64)
        self._check(self.lib.kpm_export_halo(self.h, ctypes.byref(nr), _ptr(recv), ctypes.byref(ns), _ptr(send)))
        return recv[: nr.value], send[: ns.value]

    def last_kernel(self):
        return self.lib.kpm_last_kernel(self.h).decode()

    def sell_info(self):
        info = kpm_sell_info()
        self._check(self.lib.kpm_get_sell_info(self.h, ctypes.byref(info)))
        return info

    def export_sell(self):
        info = self.sell_info()
        val = np.zeros(info.n_slots, dtype=np.complex128)
        col = np.zeros(info.n_slots, dtype=np.int32)
        cptr = np.zeros(info.n_chunks + 1, dtype=np.int64)
        perm = np.zeros(info.n_loc, dtype=np.int32)
        halo = np.zeros(max(info.n_halo, 1), dtype=np.int64)
        self._check(self.lib.kpm_export_sell(self.h, _ptr(val), _ptr(col), _ptr(cptr), _ptr(perm), _ptr(halo)))
        return dict(val=val, col=col, cptr=cptr, perm=perm, halo=halo[: info.n_halo], n_pad=info.n_pad)

    def close(self):
        if getattr(self, "h", None):
            self.lib.kpm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
