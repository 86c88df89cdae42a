"""Trace the fullest cell column per species over the first steps of a bench
configuration (status word MAX_COUNT) and the store's frames per super cell:
shows when, and why, a store would grow during stepping.

    python tools/occupancy_trace.py --config c2 --steps 80
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=80)
    a = ap.parse_args()
    import torch
    import bench
    from paper_1606_02862_b200 import _lib
    from paper_1606_02862_b200.pic import init_khi
    p, seed = bench.make_params(a.config)
    sim = init_khi(p, seed=seed, validate=False, rng="device")
    print("frames", [st.frames_per_sc for st in sim.stores], flush=True)
    for t in range(a.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim.step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        st = sim._read_status()
        print(t, "%.2f ms" % dt, "max", [int(st[i, _lib.ST_MAX_COUNT]) for i in range(len(sim.stores))],
              "frames", [s.frames_per_sc for s in sim.stores], flush=True)


if __name__ == "__main__":
    main()
