"""Render the per-case parity table (profiles/r02_parity.md) from the JSON
lines the GPU tests append to $KWB_PARITY_LOG (tests/parity_util.record).

    python tools/parity_table.py gpurun_out/parity_r02c.jsonl > profiles/r02_parity.md
"""
import collections
import json
import sys


def main(path):
    rows = [json.loads(l) for l in open(path)]
    by = collections.OrderedDict()
    for r in rows:
        by.setdefault((r["case"], r["kind"]), []).append(r)
    print("| case | kind | worst J rel-L2 | worst E/B rel-L2 | reference order spread (J) | bar | worst err / bar |")
    print("|---|---|---|---|---|---|---|")
    for (case, kind), rs in by.items():
        j = [r for r in rs if r["field"].startswith("J")]
        eb = [r for r in rs if r["field"][0] in "EB"]
        other = [r for r in rs if r not in j and r not in eb]
        def ratio(r):
            return r["err"] / r["tol"] if r["tol"] else (0.0 if r["err"] == 0 else float("inf"))
        w = max(rs, key=ratio)
        fj = f"{max(r['err'] for r in j):.2e}" if j else "-"
        feb = f"{max(r['err'] for r in eb):.2e}" if eb else "-"
        if other and not j:
            fj = f"{other[0]['field']} {other[0]['err']:.2e}"
        sp = max((r.get("spread", 0.0) for r in j), default=0.0)
        tol = sorted({r["tol"] for r in rs})
        tols = "/".join(f"{t:.1e}" for t in tol)
        print(f"| {case} | {kind} | {fj} | {feb} | {sp:.1e} | {tols} | {ratio(w):.2f} |")


if __name__ == "__main__":
    main(sys.argv[1])
