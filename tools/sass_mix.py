"""Static SASS instruction mix of every kernel instance in libkwb200.so
(cuobjdump -sass), for the profiles/ record: total instructions and the
counts that back the design claims -- spills (LDL/STL), TMA (UTMALDG /
UTMAREDG), cp.async (LDGSTS), fp64 (DFMA/DMUL/DADD), shared atomics (ATOMS),
global reductions (RED), packed fp32 (FFMA2/FMUL2/FADD2), MUFU.

    python tools/sass_mix.py paper_1606_02862_b200/libkwb200.so > profiles/r02_sass_mix.md
"""
import collections
import re
import subprocess
import sys

KEYS = ("LDL", "STL", "UTMALDG", "UTMAREDG", "LDGSTS", "DFMA", "DMUL", "DADD", "DSETP", "ATOMS",
        "RED", "REDG", "FFMA2", "FMUL2", "FADD2", "FFMA", "MUFU", "LDS", "STS", "BAR", "WARPSYNC",
        "F2F", "SHFL")


def demangle(n):
    try:
        return subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    except Exception:
        return n


def main(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    fn = None
    counts = collections.OrderedDict()
    for ln in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            fn = m.group(1)
            counts[fn] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]*)?", ln)
        if m and fn:
            op = m.group(2)
            counts[fn]["total"] += 1
            counts[fn][op] += 1
    print("| kernel | SASS | " + " | ".join(KEYS) + " |")
    print("|---|---|" + "---|" * len(KEYS))
    for fn, c in counts.items():
        name = demangle(fn)
        if "kwb::" not in name:
            continue
        short = re.sub(r"\(.*", "", name).replace("kwb::", "").replace("void ", "")
        short = short.replace("float", "f32").replace("double", "f64").replace(" ", "")
        print(f"| `{short}` | {c['total']} | " + " | ".join(str(c[k]) for k in KEYS) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
