"""Compile the in-tree sm_100a library libkpm.so (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libkpm.so")
SOURCES = ["kernels.cu", "kpm_abi.cu", "sell_build.cpp", "halo_plan.cpp", "plan_abi.cpp", "chunk_order.cpp", "dos.cpp", "sell_device.cu", "naive.cu", "hermitian.cpp"]
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand == "nvcc" or os.path.exists(cand):
            return cand
    return "nvcc"


def _nccl_dir() -> str:
    """NCCL headers + library of the image (the pip nvidia-nccl package torch itself loads)."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl.h not found (expected site-packages/nvidia/nccl)")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "kpm.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    nccl = _nccl_dir()
    cmd = [_nvcc(), *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-Xptxas", "-v", f"-I{os.path.join(ROOT, 'include')}", f"-I{nccl}/include", "-o", tmp]
    cmd += [os.path.join(CSRC, s) for s in SOURCES]
    cmd += [f"-L{nccl}/lib", "-l:libnccl.so.2", f"-Xlinker=-rpath={nccl}/lib"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    with open(os.path.join(PKG, "build.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libkpm.so (see paper_1410_5242_b200/build.log)")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
