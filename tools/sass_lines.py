"""Static SASS instruction counts of one kernel, bucketed by source line
ranges (nvdisasm -g -c line info).  Usage:
    python tools/sass_lines.py CUBIN KERNEL_MANGLED [ranges.json]
Prints per (file:line) counts and an opcode mix."""
import collections
import re
import subprocess
import sys


def parse(cubin, kernel):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    lines = out.split("\n")
    start = None
    for i, l in enumerate(lines):
        if l.startswith(".text." + kernel + ":"):
            start = i
            break
    if start is None:
        raise SystemExit("kernel not found")
    cur = ("?", 0)
    recs = []
    for l in lines[start + 1:]:
        if l.startswith(".text.") or l.startswith(".section"):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", l)
        if m:
            recs.append((int(m.group(1), 16), cur, m.group(3)))
    return recs


if __name__ == "__main__":
    recs = parse(sys.argv[1], sys.argv[2])
    by = collections.Counter(r[1] for r in recs)
    for (f, ln), n in sorted(by.items()):
        print(f"{f}:{ln} {n}")
    ops = collections.Counter(r[2].split(".")[0] for r in recs)
    print("total", len(recs))
    print(ops.most_common(40))
