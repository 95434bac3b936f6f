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
