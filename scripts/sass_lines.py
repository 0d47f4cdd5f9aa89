"""Attribute ncu per-instruction metrics to source lines of the kernel body.

    python scripts/sass_lines.py --so paper_2102_05297_b200/libct_b200.so \
        --kernel _ZN2ct16k_profile_searchILi128EEEvNS_10SearchArgsE \
        --rep gpurun_out/x_search_full.ncu-rep --file ct_search.cuh

The ncu source page lists the kernel's SASS in address order with warp-stall
samples and executed instructions; nvdisasm -gi of the same cubin gives each
instruction's (file, line) with its inlining chain.  Every instruction is
charged to the outermost frame inside --file (the kernel body line that
called the inlined helper), and the totals are printed per line.
"""

import argparse
import csv
import io
import os
import re
import subprocess
import tempfile
from collections import defaultdict

INNERMOST = False


def sass_lines(so, kernel, file_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, check=True,
                   capture_output=True)
    cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    text = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cubin)],
                          capture_output=True, text=True, check=True).stdout
    start = text.index(f".text.{kernel}:")
    end = text.find("//---------------------", start)
    body = text[start:end if end > 0 else len(text)]
    loc = None
    out = {}
    pat = re.compile(r'//## File "([^"]+)", line (\d+)(.*)')
    for line in body.splitlines():
        m = pat.search(line)
        if m:
            frames = [(m.group(1), int(m.group(2)))]
            frames += [(f, int(l)) for f, l in re.findall(r'inlined at "([^"]+)", line (\d+)',
                                                          m.group(3))]
            inside = [l for f, l in frames if file_sub in f]
            if INNERMOST:
                loc = inside[0] if inside else frames[-1][1]
            else:
                loc = inside[-1] if inside else frames[-1][1]
            continue
        a = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
        if a:
            out[int(a.group(1), 16)] = loc
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", required=True)
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--rep", required=True)
    ap.add_argument("--file", default="ct_search.cuh")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--innermost", action="store_true",
                    help="charge each instruction to its innermost line inside --file")
    a = ap.parse_args()
    global INNERMOST
    INNERMOST = a.innermost
    lines = sass_lines(a.so, a.kernel, a.file)
    page = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source",
                           "sass"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(page)))
    hdr, data = rows[1], rows[2:]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_e = hdr.index("Instructions Executed")
    base = int(data[0][0], 16)
    agg_s, agg_e = defaultdict(float), defaultdict(float)
    for r in data:
        off = int(r[0], 16) - base
        ln = lines.get(off)
        agg_s[ln] += float(r[i_s] or 0)
        agg_e[ln] += float(r[i_e] or 0)
    ts, te = sum(agg_s.values()) or 1, sum(agg_e.values()) or 1
    src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                            "paper_2102_05297_b200", "csrc", a.file)).read().splitlines()
    print(f"{'line':>5} {'stall%':>7} {'inst%':>7}  source")
    for ln in sorted(agg_s, key=lambda k: -(agg_s[k] / ts + agg_e[k] / te))[:a.top]:
        text = src[ln - 1].strip()[:80] if isinstance(ln, int) and 0 < ln <= len(src) else ""
        print(f"{str(ln):>5} {agg_s[ln] / ts * 100:7.2f} {agg_e[ln] / te * 100:7.2f}  {text}")


if __name__ == "__main__":
    main()
