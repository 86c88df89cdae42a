#!/usr/bin/env python
"""Attribute an ncu SASS source page to CUDA source lines.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX CUBIN [top]

Joins the per-instruction counters of `ncu --page source --print-source=sass`
(instructions executed, warp-stall samples) with the line table of the same
kernel in CUBIN (`nvdisasm -g`, needs -lineinfo), and prints the hottest
source lines.  The CUBIN must be the one that was profiled.
"""

import collections
import csv
import io
import re
import subprocess
import sys


def sass_lines(cubin, kernel_regex):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    fn = None
    cur_line = None
    table = {}
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
        if m:
            cur_line = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and fn and re.search(kernel_regex, fn):
            table.setdefault(fn, {})[int(m.group(1), 16)] = cur_line
    return table


def main():
    rep, kre, cubin = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4].isdigit() else 40
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ai, ie, ws = hdr.index("Address"), hdr.index("Instructions Executed"), \
        hdr.index("Warp Stall Sampling (All Samples)")
    recs = [r for r in rows[2:] if len(r) == len(hdr)]
    base = int(recs[0][ai], 16)
    tables = sass_lines(cubin, kre)
    if not tables:
        sys.exit("kernel not found in cubin")
    # pick the function whose size matches the profiled instruction count
    fn, table = min(tables.items(), key=lambda kv: abs(len(kv[1]) - len(recs)))
    agg = collections.defaultdict(lambda: [0, 0])
    tot = [0, 0]
    for r in recs:
        off = int(r[ai], 16) - base
        line = table.get(off, "?")
        a = agg[line]
        a[0] += int(r[ie] or 0)
        a[1] += int(r[ws] or 0)
        tot[0] += int(r[ie] or 0)
        tot[1] += int(r[ws] or 0)
    print(f"{fn}: {len(recs)} SASS instructions, {tot[0]:.3e} executed, {tot[1]} stall samples")
    key = 0 if "--by-inst" in sys.argv else 1
    for line, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
        print(f"{line:28s} inst {100 * n / max(tot[0], 1):5.1f}%  stall {100 * s / max(tot[1], 1):5.1f}%")


if __name__ == "__main__":
    main()
