"""Wall-clock phases of one z-slab step (DecomposedSimulation, G slabs in
this process over LoopbackTransport), against the single-domain step on the
same global problem: where the decomposition overhead goes.

    python tools/zslab_breakdown.py [--config c2] [--slabs 1] [--steps 10]
"""

import argparse
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--slabs", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    import torch
    import bench
    from paper_1606_02862_b200.pic.decomp import DecomposedSimulation, LoopbackTransport
    p, seed = bench.make_params(a.config)
    dec = DecomposedSimulation(p, a.slabs, list(range(a.slabs)), LoopbackTransport())
    dec.init_khi_slabs(seed, rng="device")
    for _ in range(3):
        dec.step()
    dec.check_status()
    torch.cuda.synchronize()
    phases = collections.defaultdict(float)

    def timed(name, fn):
        def w(*args, **kw):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = fn(*args, **kw)
            torch.cuda.synchronize()
            phases[name] += time.perf_counter() - t0
            return r
        return w

    for name in ("_exchange_j", "_exchange_particles", "_exchange_e_top", "_exchange_guards"):
        setattr(dec, name, timed(name, getattr(dec, name)))
    for sim in dec.locals.values():
        sim.advance_particles = timed("advance_particles", sim.advance_particles)
        sim.faraday_half = timed("faraday_half", sim.faraday_half)
        sim.ampere = timed("ampere", sim.ampere)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        dec.step()
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) / a.steps * 1e3
    print(f"{a.config} G={a.slabs}: {tot:.3f} ms/step wall (phases synchronised)")
    for k, v in sorted(phases.items(), key=lambda kv: -kv[1]):
        print(f"  {k:22s} {v / a.steps * 1e3:8.3f} ms/step")


if __name__ == "__main__":
    main()
