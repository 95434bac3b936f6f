"""Bottleneck experiment: time the default sweep with parts of the work removed (wrong
results; timing only).  exp/libkpm_eN.so is libkpm.so built from kernels.cu with
scripts/exp_bottleneck.patch applied and -DKPM_EXP=N: 1 = no TMA copies of the non-own V
runs, 2 = no shared-memory V gathers, 3 = both; N = 0 is the product library.

    python scripts/exp_bottleneck.py --build      # here (nvcc), writes exp/libkpm_e{0..3}.so
    python scripts/exp_bottleneck.py 2            # on the GPU box
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402


def build_libs():
    import shutil
    import subprocess
    import tempfile

    from paper_1410_5242_b200 import build as b
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    os.makedirs(os.path.join(root, "exp"), exist_ok=True)
    tmp = tempfile.mkdtemp()
    shutil.copytree(os.path.join(root, "paper_1410_5242_b200", "csrc"), os.path.join(tmp, "paper_1410_5242_b200", "csrc"))
    shutil.copytree(os.path.join(root, "include"), os.path.join(tmp, "include"))
    subprocess.run(["patch", "-p1", "-i", os.path.join(root, "scripts", "exp_bottleneck.patch")], cwd=tmp, check=True)
    nccl = b._nccl_dir()
    for e in [int(x) for x in os.environ.get("EXP_LIST", "0,1,2,3").split(",")]:
        cmd = [b._nvcc(), *b.GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
               f"-DKPM_EXP={e}", f"-I{os.path.join(root, 'include')}", f"-I{nccl}/include",
               "-o", os.path.join(root, "exp", f"libkpm_e{e}.so")]
        cmd += [os.path.join(tmp, "paper_1410_5242_b200", "csrc", s) for s in b.SOURCES]
        cmd += [f"-L{nccl}/lib", "-l:libnccl.so.2", f"-Xlinker=-rpath={nccl}/lib"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stderr[-3000:])


def main():
    if sys.argv[1] == "--build":
        build_libs()
        return
    import paper_1410_5242_b200 as kpm
    e = sys.argv[1]
    kpm.LIB_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "exp", f"libkpm_e{e}.so")
    lat = Lattice(200, 100, 40)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    for R in (8, 16, 32):
        with kpm.KpmContext() as ctx:
            ctx.set_matrix(rp, col, val, a, b)
            ctx.moments(200, R, SEED, want_eta=False)
            best = 1e9
            for _ in range(3):
                ctx.moments(400, R, SEED, want_eta=False)
                best = min(best, ctx.last_timing()[1])
            print(json.dumps(dict(exp=int(e), R=R, kernel=ctx.last_kernel(), sweep_ms=best)), flush=True)


if __name__ == "__main__":
    main()
