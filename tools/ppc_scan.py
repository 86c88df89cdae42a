"""Advance-launch time against particles per cell on a fixed grid (C4
physics: 128^3 thermal electrons, TSC, fp32): separates the per-super-cell
fixed cost (staging, sweeps, flush, barriers) from the per-particle cost.

    python tools/ppc_scan.py [--ppc 8 16 32 64]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ppc", type=int, nargs="+", default=[8, 16, 32, 64])
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_1606_02862_b200 import _lib
    from paper_1606_02862_b200.pic import SimParams, Species, init_khi
    import paper_1606_02862_b200.pic.sim as simmod
    rows = []
    for ppc in a.ppc:
        p = SimParams(cells=(128, 128, 128), species=(Species("electron", -1.0, 1.0, 1.0 / ppc),),
                      particles_per_cell=ppc, dtype=np.float32, shape="tsc",
                      stream_velocity=0.0, perturbation=0.0, thermal_u=0.05)
        sim = init_khi(p, seed=4, validate=False, rng="device")
        sim.use_graphs = False
        for _ in range(10):
            sim.enqueue_step()
        sim.check_status()
        ev = []
        orig = _lib.call

        def timed(name, *args):
            if name == "kwb_particles_advance":
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                orig(name, *args)
                e1.record()
                ev.append((e0, e1))
            else:
                orig(name, *args)
        simmod._lib.call = timed
        for _ in range(a.steps):
            sim.enqueue_step()
        torch.cuda.synchronize()
        simmod._lib.call = orig
        sim.check_status()
        ms = sum(e0.elapsed_time(e1) for e0, e1 in ev) / len(ev)
        n = sim.census()
        rows.append((ppc, n, ms))
        print(f"ppc {ppc:3d}: {n:12d} particles, advance {ms:.3f} ms, {n / ms / 1e6:.2f} M/ms", flush=True)
        del sim
        torch.cuda.empty_cache()
    x = np.array([r[1] for r in rows], dtype=float)
    y = np.array([r[2] for r in rows])
    A = np.vstack([np.ones_like(x), x]).T
    c0, c1 = np.linalg.lstsq(A, y, rcond=None)[0]
    print(f"fit: advance = {c0:.3f} ms + {c1 * 1e6:.4f} ms per M particles")


if __name__ == "__main__":
    main()
