"""Cost of validate=True (on-device rho, continuity residual and Gauss drift
every step) against validate=False, same config, Simulation.step().

    python tools/validate_cost.py [--config c2] [--steps 10]
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    import torch
    import bench
    from paper_1606_02862_b200.pic import init_khi
    p, seed = bench.make_params(a.config)
    for validate in (False, True):
        sim = init_khi(p, seed=seed, validate=validate, rng="device")
        for _ in range(3):
            sim.step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            sim.step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / a.steps * 1e3
        extra = f", residual {sim.last_residual:.2e}, gauss drift {sim.last_gauss_drift:.2e}" \
            if validate else ""
        print(f"{a.config} validate={validate}: {dt:.3f} ms/step{extra}", flush=True)
        del sim
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
