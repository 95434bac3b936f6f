"""Summarise ncu captures from gpurun_out/ into profiles/ (run here, no GPU needed).

    python scripts/ncu_summary.py --round r01 --launches gpurun_out/launches.csv \
        --full gpurun_out/full_r32.ncu-rep:C3/R32 gpurun_out/full_r8.ncu-rep:C3/R8 ...
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
    "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
]


def raw(rep):
    """Metrics of an ncu report (.ncu-rep) or of its `ncu -i ... --page raw --csv` export (.csv)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


def stall_top(rep, k=8):
    d = raw(rep)
    tot = [(float(v[1].replace(",", "")), n) for n, v in d.items()
           if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")
           and v[1].replace(",", "").replace(".", "").isdigit()]
    s = sum(x for x, _ in tot) or 1.0
    tot.sort(reverse=True)
    return {n.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(100 * x / s, 1) for x, n in tot[:k]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--launches")
    ap.add_argument("--full", nargs="*", default=[])
    args = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    if args.launches:
        rows = [r for r in csv.reader(open(args.launches)) if len(r) > 5]
        hdr = rows[0]
        ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        t, n = defaultdict(float), defaultdict(int)
        for r in rows[1:]:
            ms = float(r[iv].replace(",", "")) * UNIT.get(r[iu], 1.0)
            name = r[ik].split("(")[0].replace("void ", "").replace("unnamed>::", "")
            t[name] += ms
            n[name] += 1
        tot = sum(t.values())
        lines = [f"# launch list ({args.launches}): {sum(n.values())} launches, ncu --metrics gpu__time_duration.sum "
                 "--clock-control none (cold-cache, serialised: compare shares)",
                 f"{'kernel':48s} {'launches':>8s} {'total ms':>10s} {'avg ms':>9s} {'share':>7s}"]
        for k in sorted(t, key=lambda k: -t[k]):
            lines.append(f"{k:48s} {n[k]:8d} {t[k]:10.3f} {t[k] / n[k]:9.4f} {100 * t[k] / tot:6.2f}%")
        open(os.path.join(prof, f"{args.round}_launches.txt"), "w").write("\n".join(lines) + "\n")
        import shutil

        shutil.copy(args.launches, os.path.join(prof, f"{args.round}_launches.csv"))
        print("\n".join(lines))
    traffic_path = os.path.join(prof, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    full_path = os.path.join(prof, f"{args.round}_ncu_full.json")
    summary = json.load(open(full_path)) if os.path.exists(full_path) else {}  # merge: captures come per call
    for spec in args.full:
        rep, tag = spec.split(":")
        d = raw(rep)
        vals = {k: d[k][1] + " " + d[k][0] for k in KEYS if k in d}
        vals["stall_top_pct"] = stall_top(rep)
        summary[tag] = vals

        def num(key, scale):
            u, v = d[key]
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            return float(v.replace(",", "")) * mult / scale

        dram = num("dram__bytes_read.sum", 1) + num("dram__bytes_write.sum", 1)
        lattice, r = tag.split("/")
        traffic[f"{lattice}/{r}"] = dram
        vals["dram_bytes_per_launch"] = dram
        smem = float(d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"][1].replace(",", ""))
        traffic[f"{lattice}/{r}/smem_wavefronts"] = smem
    if args.full:
        json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
        with open(full_path, "w") as f:
            json.dump(summary, f, indent=1)
        print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
