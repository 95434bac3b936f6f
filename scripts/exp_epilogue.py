"""Epilogue / index experiment (timing only, wrong results): the default tiled sweep with
parts of its shared-memory traffic removed, to size candidate optimisations before
building them.  Bits of -DKPM_EXP:
   4  epilogue takes V_i from registers instead of the shared-memory own row
   8  no old-W tile (neither its TMA copy nor its shared-memory read)
  16  no lcol loads in the gather loop (each entry gathers row (k + j) mod 32 of the tile)
N = 0 is the product kernel.  exp/libkpm_xN.so are built here; run on the GPU box:

    python scripts/exp_epilogue.py --build 0,4,8,16,28
    python scripts/exp_epilogue.py 4
"""
import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402

EDITS = [
    ("const double2 vi = sV[kr * R + col];",
     "const double2 vi = (KPM_EXP & 4) ? make_double2(u[cc].y, u[cc].x) : sV[kr * R + col];"),
    ("const double2 wo = WS ? sW[kr * R + col] : wreg[cc];",
     "const double2 wo = (KPM_EXP & 8) ? make_double2(0.5 * u[cc].x, u[cc].y) : (WS ? sW[kr * R + col] : wreg[cc]);"),
    ("const uint32_t total = __shfl_sync(0xffffffffu, W_TILE ? cur.x : cur.y, 0);",
     "const uint32_t total = __shfl_sync(0xffffffffu, (W_TILE && !(KPM_EXP & 8)) ? cur.x : cur.y, 0);"),
    ("if (W_TILE || base != 1) {", "if ((W_TILE && !(KPM_EXP & 8)) || base != 1) {"),
    ("li[uu] = sl[(j + uu) * kC] * R;", "li[uu] = (KPM_EXP & 16) ? ((kr + j + uu) & 31) * R : sl[(j + uu) * kC] * R;"),
    ("const int li = sl[j * kC] * R;", "const int li = (KPM_EXP & 16) ? ((kr + j) & 31) * R : sl[j * kC] * R;"),
]


def build_libs(exps):
    from paper_1410_5242_b200 import build as b
    os.makedirs(os.path.join(ROOT, "exp"), exist_ok=True)
    tmp = tempfile.mkdtemp()
    src = os.path.join(tmp, "pkg", "csrc")
    shutil.copytree(os.path.join(ROOT, "paper_1410_5242_b200", "csrc"), src)
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
    k = os.path.join(src, "kernels.cu")
    s = open(k).read()
    for old, new in EDITS:
        assert old in s, old
        s = s.replace(old, new)
    open(k, "w").write("#ifndef KPM_EXP\n#define KPM_EXP 0\n#endif\n" + s)
    nccl = b._nccl_dir()
    for e in exps:
        cmd = [b._nvcc(), *b.GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
               f"-DKPM_EXP={e}", f"-I{os.path.join(ROOT, 'include')}", f"-I{nccl}/include",
               "-o", os.path.join(ROOT, "exp", f"libkpm_x{e}.so")]
        cmd += [os.path.join(src, f) for f in b.SOURCES]
        cmd += [f"-L{nccl}/lib", "-l:libnccl.so.2", f"-Xlinker=-rpath={nccl}/lib"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stderr[-3000:])


def main():
    if sys.argv[1] == "--build":
        build_libs([int(x) for x in sys.argv[2].split(",")])
        return
    import paper_1410_5242_b200 as kpm
    e = sys.argv[1]
    kpm.LIB_PATH = os.path.join(ROOT, "exp", f"libkpm_x{e}.so")
    lat = Lattice(200, 100, 40)
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    for R in [int(r) for r in os.environ.get("EXP_R", "8,16,32").split(",")]:
        with kpm.KpmContext() as ctx:
            ctx.set_matrix(rp, col, val, a, b)
            ctx.moments(200, R, SEED, want_eta=False)
            best = 1e9
            for _ in range(3):
                ctx.moments(400, R, SEED, want_eta=False)
                best = min(best, ctx.last_timing()[1])
            print(json.dumps(dict(exp=e, R=R, kernel=ctx.last_kernel(), sweep_ms=best)), flush=True)


if __name__ == "__main__":
    main()
