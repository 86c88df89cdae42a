"""A/B timing of experiment builds on one GPU: runs bench.py with each
library (KWB_LIB_PATH) in interleaved order and prints median step time and
mean advance-launch time per library.

    python tools/ab.py [--config c2] [--rounds 2] lib_a.so lib_b.so ...
"""

import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("libs", nargs="+", help="library paths; LIB@VAR=VAL sets an env var for that arm")
    a = ap.parse_args()
    res = {lib: [] for lib in a.libs}
    for r in range(a.rounds):
        for lib in a.libs:
            path, _, kv = lib.partition("@")
            env = dict(os.environ, KWB_LIB_PATH=os.path.abspath(path))
            if kv:
                k, _, v = kv.partition("=")
                env[k] = v
            out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", a.config,
                                  "--steps", str(a.steps), "--warmup", str(a.warmup), "--no-cpu"],
                                 capture_output=True, text=True, env=env, cwd=ROOT)
            try:
                d = json.loads(out.stdout.strip().splitlines()[-1])
            except Exception:
                print(lib, "FAILED", out.stderr[-2000:], flush=True)
                continue
            med = d["ms_per_step_quartiles"][2]
            adv = d["roofline"]["mean_launch_ms"]
            res[lib].append((med, adv))
            print(f"round {r} {os.path.basename(lib):32s} median step {med:7.3f} ms  "
                  f"advance {adv:6.3f} ms", flush=True)
    for lib, v in res.items():
        if v:
            print(f"SUMMARY {os.path.basename(lib):32s} step {statistics.median(x[0] for x in v):7.3f} "
                  f"advance {statistics.median(x[1] for x in v):6.3f}")


if __name__ == "__main__":
    main()
