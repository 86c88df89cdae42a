"""Wall-clock cost of the synchronous Simulation.step() (two host syncs per
cycle, the reference's semantics) against the asynchronous enqueue_step()
(lagged status), same state, same number of steps.

    python tools/sync_step_cost.py [--config c2] [--steps 20]
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    import torch
    import bench
    from paper_1606_02862_b200.pic import init_khi
    p, seed = bench.make_params(a.config)
    sim = init_khi(p, seed=seed, validate=False, rng="device")
    for _ in range(3):
        sim.enqueue_step()
    sim.check_status()
    torch.cuda.synchronize()
    for name, fn in (("enqueue_step", sim.enqueue_step), ("step", sim.step),
                     ("enqueue_step", sim.enqueue_step), ("step", sim.step)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            fn()
        sim.check_status()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / a.steps * 1e3
        print(f"{name:14s} {dt:8.3f} ms/step wall", flush=True)


if __name__ == "__main__":
    main()
