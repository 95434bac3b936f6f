"""CPU tests of the boundary: the library builds for sm_100a, loads without a GPU and
exports every entry point include/kpm.h declares; the binding fails loudly without it."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1410_5242_b200 import build

    build.build()
    import paper_1410_5242_b200 as pkg

    return pkg.load_library()


def header_functions():
    text = open(os.path.join(ROOT, "include", "kpm.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kpm_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported(lib):
    names = header_functions()
    assert "kpm_create" in names and "kpm_moments" in names and "kpm_destroy" in names
    for n in names:
        assert hasattr(lib, n), n
    import paper_1410_5242_b200 as pkg

    assert sorted(pkg.ABI_SYMBOLS) == names


def test_library_is_sm100a(lib):
    import paper_1410_5242_b200 as pkg

    out = subprocess.run(["cuobjdump", "--list-elf", pkg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_create_fails_loudly(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1410_5242_b200 as pkg

    with pytest.raises(pkg.KpmError):
        pkg.KpmContext(device=0)


def test_header_compiles_as_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "kpm.h"\nint main(void){kpm_ctx* c=0; kpm_destroy(c); return 0;}\n')
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-c", f"-I{ROOT}/include", str(src), "-o",
                    str(tmp_path / "t.o")], check=True)


def build_c_demo(tmp_path):
    """Compile tests/c_abi/kpm_c_demo.c (plain C99) against include/kpm.h and link libkpm.so."""
    import paper_1410_5242_b200 as pkg

    libdir = os.path.dirname(pkg.LIB_PATH)
    exe = tmp_path / "kpm_c_demo"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "c_abi", "kpm_c_demo.c"), "-o", str(exe), f"-L{libdir}", "-l:libkpm.so",
                    f"-Wl,-rpath,{libdir}"], check=True)
    return exe


def write_csr(path, rp, col, val):
    import numpy as np

    with open(path, "wb") as f:
        np.array([len(rp) - 1, len(col)], dtype=np.int64).tofile(f)
        np.asarray(rp, dtype=np.int64).tofile(f)
        np.asarray(col, dtype=np.int64).tofile(f)
        np.asarray(val, dtype=np.complex128).tofile(f)


def test_c_caller_links_and_fails_loudly_without_gpu(lib, tmp_path):
    """A plain-C program links libkpm.so and calls the ABI; without a GPU kpm_create returns an
    error status with a message (no CPU fallback)."""
    import torch

    from workloads.ti_lattice import Lattice, generate_csr

    exe = build_c_demo(tmp_path)
    lat = Lattice(4, 4, 4)
    rp, col, val = generate_csr(lat)
    write_csr(tmp_path / "h.bin", rp, col, val)
    r = subprocess.run([str(exe), str(tmp_path / "h.bin"), "0.1", "0", "16", "2", "7"], capture_output=True, text=True)
    if torch.cuda.is_available():
        assert r.returncode == 0 and len(r.stdout.split()) == 16
    else:
        assert r.returncode == 2 and "kpm_create" in r.stderr, (r.returncode, r.stderr)
