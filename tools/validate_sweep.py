"""validate=True on every bench config for a few steps: the on-device
continuity residual and Gauss drift stay inside the reference's bars
(1e-12 / 1e-13 float64, 1e-6 float32) at full size.

    python tools/validate_sweep.py [--steps 5]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--configs", nargs="+",
                    default=["c1", "c1_tsc", "c2", "c2_f64", "c3", "c4_cic", "c4_tsc", "c4_pcs", "c5"])
    a = ap.parse_args()
    import numpy as np
    import torch
    import bench
    from paper_1606_02862_b200.pic import init_khi
    ok = True
    for cfg in a.configs:
        p, seed = bench.make_params(cfg)
        sim = init_khi(p, seed=seed, validate=True, rng="device")
        worst_r = worst_g = 0.0
        for _ in range(a.steps):
            sim.step()
            worst_r = max(worst_r, sim.last_residual)
            worst_g = max(worst_g, sim.last_gauss_drift)
        lim = 1e-12 if p.dtype == np.float64 else 1e-6
        glim = 1e-13 if p.dtype == np.float64 else 1e-6
        good = worst_r <= lim and worst_g <= glim
        ok &= good
        print(f"{cfg:8s} residual {worst_r:.2e} (<= {lim:g}) gauss drift {worst_g:.2e} "
              f"(<= {glim:g}) {'ok' if good else 'FAIL'}", flush=True)
        del sim
        torch.cuda.empty_cache()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
