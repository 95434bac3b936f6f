"""The paper's bottleneck analysis on a B200 (Figs. 8-9): plain SpMMV, augmented
SpMMV without dots and the fully augmented SpMMV, block widths R = 1..32, C3 lattice.

    python scripts/fig9_kernels.py --out gpurun_out/fig9_time.json          # device timing
    ncu --metrics <METRICS> --clock-control none -k regex:aug_spmmv_tiled --csv \
        --log-file gpurun_out/fig9_ncu.csv python scripts/fig9_kernels.py --ncu
    python scripts/fig9_kernels.py --summarise gpurun_out/fig9_time.json gpurun_out/fig9_ncu.csv \
        > profiles/r01_fig9.json                                             # here, no GPU

--ncu runs each (kind, R) exactly once (one sweep, no warm-up) in the fixed order of CONFIGS,
so the i-th captured launch is CONFIGS[i].
"""
import argparse
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from workloads.ti_lattice import SEED, Lattice, gershgorin, generate_csr, scale_factors  # noqa: E402

KINDS = ["spmmv", "aug_nodot", "aug"]
WIDTHS = [1, 2, 4, 8, 16, 32]
CONFIGS = [(k, r) for r in WIDTHS for k in KINDS]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
           "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
           "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]
UNIT = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def alg_bytes(kind, R, n, nnz):
    """Minimum HBM traffic per sweep: matrix 20 B per entry; SpMMV reads V and
    writes W (32 R N); the augmented kinds also read the old W (48 R N)."""
    return 20 * nnz + (32 if kind == "spmmv" else 48) * R * n


def run(args):
    import paper_1410_5242_b200 as kpm

    lat = Lattice(*(int(t) for t in args.lattice.split(",")))
    rp, col, val = generate_csr(lat)
    a, b = scale_factors(*gershgorin(rp, col, val))
    n, nnz = lat.n, int(rp[-1])
    rows = []
    with kpm.KpmContext() as ctx:
        ctx.set_matrix(rp, col, val, a, b)
        for kind, R in CONFIGS:
            if args.ncu:
                ctx.sweep_kernel(kind, R, SEED, n_sweeps=1)
                continue
            ctx.sweep_kernel(kind, R, SEED, n_sweeps=5)  # warm-up
            ms, _ = ctx.sweep_kernel(kind, R, SEED, n_sweeps=args.sweeps)
            by = alg_bytes(kind, R, n, nnz)
            row = dict(kind=kind, R=R, kernel=ctx.last_kernel(), ms=ms, alg_bytes=by, alg_gbs=by / ms / 1e6,
                       alg_frac=by / ms / 1e6 / 6450.0)
            if kind == "aug":
                row["gflops"] = R * (8 * nnz + 34 * n) / ms / 1e6
            rows.append(row)
            print(json.dumps(row), flush=True)
    if not args.ncu:
        json.dump(dict(lattice=args.lattice, n=n, nnz=nnz, sweeps=args.sweeps, rows=rows), open(args.out, "w"), indent=1)


def summarise(time_json, ncu_csv):
    t = json.load(open(time_json))
    rows = [r for r in csv.reader(open(ncu_csv)) if len(r) > 5]
    hdr = rows[0]
    iid, ik, im, iu, iv = (hdr.index(h) for h in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    per = {}
    for r in rows[1:]:
        if "aug_spmmv_tiled" not in r[ik]:
            continue
        per.setdefault(int(r[iid]), {})[r[im]] = float(r[iv].replace(",", "")) * UNIT.get(r[iu], 1.0)
    launches = [per[i] for i in sorted(per)]
    assert len(launches) == len(CONFIGS), (len(launches), len(CONFIGS))
    out = []
    timing = {(r["kind"], r["R"]): r for r in t["rows"]}
    for (kind, R), m in zip(CONFIGS, launches):
        dur = m["gpu__time_duration.sum"]
        dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        l2 = m["lts__t_bytes.sum"]
        l2sm = m["l1tex__m_xbar2l1tex_read_bytes.sum"]
        smem = m["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"] * 128
        tm = timing[(kind, R)]
        out.append(dict(kind=kind, R=R, kernel=tm["kernel"], ms_events=tm["ms"], ms_ncu=dur * 1e3,
                        alg_gb=tm["alg_bytes"] / 1e9, omega=dram / tm["alg_bytes"],
                        volume_gb_per_vector={"dram": dram / R / 1e9, "l2": l2 / R / 1e9, "l2_to_sm": l2sm / R / 1e9,
                                              "smem_lsu": smem / R / 1e9},
                        bandwidth_tbs={"dram": dram / dur / 1e12, "l2": l2 / dur / 1e12, "l2_to_sm": l2sm / dur / 1e12,
                                       "smem_lsu": smem / dur / 1e12},
                        sm_ghz=m["sm__cycles_elapsed.avg.per_second"] / 1e9,
                        insts_per_row=m["smsp__inst_executed.sum"] / t["n"]))
    return dict(what="the paper's Figs. 8-9 bottleneck analysis on one B200: plain SpMMV, augmented SpMMV "
                     "without dots, fully augmented SpMMV (P:764-821); C3 lattice " + t["lattice"],
                timing="ms_events: CUDA events, average over the sweeps of kpm_sweep_kernel after 5 warm-up sweeps",
                ncu="one launch per (kind, R), ncu --clock-control none; volumes per block vector (÷R)",
                rows=out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lattice", default="200,100,40")
    ap.add_argument("--sweeps", type=int, default=50)
    ap.add_argument("--out", default="gpurun_out/fig9_time.json")
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--summarise", nargs=2)
    args = ap.parse_args()
    if args.summarise:
        print(json.dumps(summarise(*args.summarise), indent=1))
        return
    run(args)


if __name__ == "__main__":
    main()
