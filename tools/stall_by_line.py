"""Map ncu SASS-level warp-stall samples of one kernel to CUDA source lines.

    python tools/stall_by_line.py <report.ncu-rep> <kernel-regex> <cubin> [launch-index]

ncu's `--page source --csv` gives per-SASS-instruction samples with runtime
addresses; `nvdisasm --print-line-info` on the same cubin gives per-offset
source lines (the library is built with -lineinfo).  Offsets are taken
relative to the first instruction of the kernel in both listings.
"""
from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys


def sass_samples(rep, kernel, idx):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}", "--kernel-name-base", "demangled",
                          "--launch-skip", str(idx), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    out = []
    for r in rows[hdr_i + 1:]:
        if len(r) > si and r[0].startswith("0x"):
            out.append((int(r[0], 16), r[1].strip(), int(r[si] or 0)))
    return out


def line_map(cubin, func_regex):
    txt = subprocess.run(["nvdisasm", "--print-line-info", "-c", cubin], capture_output=True, text=True).stdout
    cur_fn, cur_line, m = None, None, {}
    for ln in txt.splitlines():
        if ln.startswith(".text.") and ln.strip().endswith(":"):
            cur_fn = ln.strip()[:-1].replace(".text.", "")
            continue
        lm = re.search(r'File "([^"]+)", line (\d+)', ln)
        if "//##" in ln and lm:
            cur_line = (lm.group(1).split("/")[-1], int(lm.group(2)))
            continue
        am = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if am and cur_fn and re.search(func_regex, cur_fn):
            m.setdefault(cur_fn, {})[int(am.group(1), 16)] = cur_line
    return m


def main():
    rep, kernel, cubin = sys.argv[1:4]
    idx = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    want = sys.argv[5] if len(sys.argv) > 5 else None  # mangled cubin function name
    smp = sass_samples(rep, kernel, idx)
    base = smp[0][0]
    maps = line_map(cubin, ".")
    # pick the function whose instruction count matches best
    fn = want if want else min(maps, key=lambda f: abs(len(maps[f]) - len(smp)))
    lm = maps[fn]
    by = collections.Counter()
    for a, _, n in smp:
        by[lm.get(a - base)] += n
    tot = sum(by.values()) or 1
    print(f"{fn}: {tot} samples")
    srcdir = sys.argv[6] if len(sys.argv) > 6 else None  # directory of the sources
    cache = {}
    for key, n in by.most_common(40):
        txt = ""
        if key and srcdir:
            f, line = key
            import os
            fp = os.path.join(srcdir, f)
            if f not in cache:
                cache[f] = open(fp).read().splitlines() if os.path.exists(fp) else []
            src = cache[f]
            txt = src[line - 1].strip()[:90] if line <= len(src) else ""
        print(f"{n:7d} {100 * n / tot:5.1f}%  {key}  {txt}")


if __name__ == "__main__":
    main()
