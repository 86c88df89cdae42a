"""Where the device time of one PIC cycle goes: CUDA events around every
C-ABI launch of enqueue_step() and around whole steps, for one bench config.
The difference between the step time and the sum of launch times is launch
gaps plus the torch memsets/copies of the step.

    python tools/step_breakdown.py [--config c2] [--steps 20]
"""

import argparse
import collections
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    import torch
    import bench
    from paper_1606_02862_b200 import _lib
    from paper_1606_02862_b200.pic import init_khi
    import paper_1606_02862_b200.pic.sim as simmod
    p, seed = bench.make_params(a.config)
    sim = init_khi(p, seed=seed, validate=False, rng="device")
    sim.use_graphs = False   # direct launches: a replayed graph hides them from the events
    stream = torch.cuda.current_stream()
    evs = []
    orig = _lib.call

    def timed(name, *args):
        if timed.on:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            orig(name, *args)
            e1.record(stream)
            evs.append((name, e0, e1))
        else:
            orig(name, *args)
    timed.on = False
    simmod._lib.call = timed
    for _ in range(3):
        sim.enqueue_step()
    sim.check_status()
    torch.cuda.synchronize()
    timed.on = True
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(a.steps):
        sim.enqueue_step()
    s1.record(stream)
    torch.cuda.synchronize()
    timed.on = False
    sim.check_status()
    step_ms = s0.elapsed_time(s1) / a.steps
    per = collections.defaultdict(list)
    for name, e0, e1 in evs:
        per[name].append(e0.elapsed_time(e1))
    tot = 0.0
    print(f"config {a.config}: {step_ms:.3f} ms/step (device, {a.steps} steps)")
    for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        ms = sum(v) / a.steps
        tot += ms
        print(f"  {name:28s} {ms:8.3f} ms/step  ({len(v) // a.steps}/step, mean {statistics.mean(v):.3f})")
    print(f"  {'sum of launches':28s} {tot:8.3f} ms/step; rest (gaps, memsets, copies) "
          f"{step_ms - tot:.3f} ms/step")


if __name__ == "__main__":
    main()
