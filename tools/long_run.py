"""Long-run stability: N enqueue steps of a bench config with a status check
every `--every` steps; prints device time per block, column capacity,
census and field energy (a thermal plasma must stay bounded).

    python tools/long_run.py [--config c2] [--steps 1000] [--every 100]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--every", type=int, default=100)
    a = ap.parse_args()
    import torch
    import bench
    from paper_1606_02862_b200.pic import init_khi
    p, seed = bench.make_params(a.config)
    sim = init_khi(p, seed=seed, validate=False, rng="device")
    n0 = sim.census()
    done = 0
    while done < a.steps:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.every):
            sim.enqueue_step()
        e1.record()
        torch.cuda.synchronize()
        st = sim.check_status()
        done += a.every
        d = sim.diagnostics()
        from paper_1606_02862_b200 import _lib
        leavers = int(st[:, _lib.ST_LEAVERS].max())   # the last step's super-cell leavers
        print(f"step {done:6d}: {e0.elapsed_time(e1) / a.every:7.3f} ms/step, frames "
              f"{[st_.frames_per_sc for st_ in sim.stores]}, census {sim.census() - n0:+d}, "
              f"leavers {leavers}, field energy {d['field_energy']:.4e}, "
              f"KE {d['kinetic_energy']:.6e}", flush=True)


if __name__ == "__main__":
    main()
