"""Summarise ncu output into a committed text file under profiles/.

    python scripts/ncu_summary.py --launches gpurun_out/launches.csv \
        --full gpurun_out/search_full.ncu-rep --out profiles/r01_search.md

launches: the `--metrics gpu__time_duration.sum --clock-control none --csv`
launch list (per-launch, cold-cache, serialised times).  full: one
`--set full` capture of the dominant kernel; the raw page is reduced to the
metrics the roofline discussion in DESIGN.md uses, and the SASS page to the
hottest instructions by warp-stall samples.
"""

import argparse
import csv
import io
import subprocess
from collections import defaultdict

RAW_METRICS = [
    ("gpu__time_duration.sum", "kernel duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("gpc__cycles_elapsed.max", "cycles elapsed"),
]


def _ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and not r[0].startswith("==")]
    hdr, data = rows[0], rows[1:]
    kn, val, unit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in data:
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[unit], 1e-3)
        agg[r[kn]].append(float(r[val].replace(",", "")) * scale)
    total = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k[:70]}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | "
                   f"{sum(v) / total * 100:.1f}% |")
    return out


def full(path):
    raw = list(csv.reader(io.StringIO(_ncu(["-i", path, "--page", "raw", "--csv"]))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    out = ["| metric | value | unit |", "|---|---|---|"]
    for m, label in RAW_METRICS:
        if m in hdr:
            i = hdr.index(m)
            out.append(f"| {label} (`{m}`) | {vals[i]} | {units[i]} |")
    sass = list(csv.reader(io.StringIO(_ncu(["-i", path, "--page", "source", "--csv",
                                             "--print-source", "sass"]))))
    h, data = sass[1], sass[2:]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    i_e = h.index("Instructions Executed")
    stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    tot_s = sum(float(r[i_s] or 0) for r in data) or 1.0
    tot_e = sum(float(r[i_e] or 0) for r in data) or 1.0
    reasons = defaultdict(float)
    for r in data:
        for i in stall_cols:
            reasons[h[i][6:]] += float(r[i] or 0)
    rs = sum(reasons.values()) or 1.0
    out += ["", "Stall reasons (share of all warp-stall samples):", "",
            "| reason | share |", "|---|---|"]
    for k, v in sorted(reasons.items(), key=lambda kv: -kv[1])[:10]:
        out.append(f"| {k} | {v / rs * 100:.1f}% |")
    out += ["", "Hottest SASS instructions (stall samples):", "",
            "| # | sample share | inst share | instruction |", "|---|---|---|---|"]
    top = sorted(range(len(data)), key=lambda k: -float(data[k][i_s] or 0))[:15]
    for k in top:
        r = data[k]
        out.append(f"| {k} | {float(r[i_s] or 0) / tot_s * 100:.2f}% | "
                   f"{float(r[i_e] or 0) / tot_e * 100:.2f}% | `{r[1].strip()[:70]}` |")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--cmd", default="")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.cmd:
        lines += ["Command:", "", "```", a.cmd, "```", ""]
    if a.launches:
        lines += ["## Launch list (`--metrics gpu__time_duration.sum --clock-control none`)", ""]
        lines += launches(a.launches) + [""]
    if a.full:
        lines += ["## `--set full` capture of the dominant kernel", ""] + full(a.full) + [""]
    with open(a.out, "w") as fh:
        fh.write("\n".join(lines))


if __name__ == "__main__":
    main()
