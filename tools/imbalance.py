"""Lane balance of the advance over a run: per step, the mean column count
(particles per cell), the mean over warps of the warp's LONGEST column (the
advance loop's trip count: one warp = 32 consecutive cells of a super cell)
and their ratio (= fraction of lanes busy in the particle loop), plus the
advance launch time of the step.

    python tools/imbalance.py [--config c2] [--steps 60] [--every 5]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--every", type=int, default=5)
    a = ap.parse_args()
    import torch
    import bench
    from paper_1606_02862_b200 import _lib
    from paper_1606_02862_b200.pic import init_khi
    import paper_1606_02862_b200.pic.sim as simmod
    p, seed = bench.make_params(a.config)
    sim = init_khi(p, seed=seed, validate=False, rng="device")
    sim.use_graphs = False
    stream = torch.cuda.current_stream()
    orig = _lib.call
    last = []

    def timed(name, *args):
        if "advance" in name:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            orig(name, *args)
            e1.record(stream)
            last.append((e0, e1))
        else:
            orig(name, *args)
    simmod._lib.call = timed
    for t in range(a.steps + 1):
        if t % a.every == 0:
            torch.cuda.synchronize()
            ms = sum(e0.elapsed_time(e1) for e0, e1 in last) if last else float("nan")
            row = [f"step {t:3d}", f"advance {ms:7.3f} ms"]
            for i, st in enumerate(sim.stores):
                cols = st.current
                n = (cols.front + cols.back).view(-1, 32).float()
                mean = n.mean().item()
                wmax = n.max(dim=1).values.mean().item()
                row.append(f"s{i}: mean {mean:6.2f} warp-max {wmax:6.2f} busy {mean / wmax:5.3f} "
                           f"max {int(n.max().item())}")
            print("  ".join(row), flush=True)
        last.clear()
        sim.enqueue_step()
    sim.check_status()


if __name__ == "__main__":
    main()
