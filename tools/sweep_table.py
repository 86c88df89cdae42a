#!/usr/bin/env python
"""Markdown table rows from the bench lines tools/config_sweep.sh leaves in
gpurun_out/sweep_<cfg>.json (one row per config, in the sweep's order).

    python tools/sweep_table.py [gpurun_out]
"""
import json
import os
import statistics
import sys

ORDER = ("c1", "c1_tsc", "c2", "c2_zslab", "c2_f64", "c3", "c4_cic", "c4_tsc", "c4_pcs", "c5")


def main():
    d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    print("| config | particles | ms/step (median) | particle-updates/s | ns/particle/cycle "
          "| advance mean (ms/launch) | roofline frac |")
    print("|---|---|---|---|---|---|---|")
    for c in ORDER:
        path = os.path.join(d, f"sweep_{c}.json")
        try:
            b = json.loads(open(path).read().strip().splitlines()[-1])
        except (OSError, ValueError, IndexError):
            print(f"| {c} | (no result) | | | | | |")
            continue
        q = b.get("ms_per_step_quartiles") or [b["ms_per_step"]] * 5
        wl = b["config"]["workload"]
        if b["config"].get("parallelism", "single") != "single":
            wl += f" [{b['config']['parallelism']}]"
        rl = b.get("roofline") or {}
        print(f"| {wl} | {b['config']['particles_per_gpu']:,} | {b['ms_per_step']:.3f} "
              f"({statistics.median(q):.3f}) | {b['value']:.3g} | {b['ns_per_particle_cycle']:.3f} "
              f"| {rl.get('mean_launch_ms', float('nan')):.3f} | {rl.get('frac', float('nan')):.3f} |")


if __name__ == "__main__":
    main()
