"""enqueue_step with and without the CUDA-graph replay, one config:
launch-bound grids (C1) gain most.

    python tools/graph_cost.py [--config c1] [--steps 200]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    import torch
    import bench
    from paper_1606_02862_b200.pic import init_khi
    p, seed = bench.make_params(a.config)
    for graphs in (False, True, False, True):
        sim = init_khi(p, seed=seed, validate=False, rng="device")
        sim.use_graphs = graphs
        for _ in range(5):
            sim.enqueue_step()
        sim.check_status()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.steps):
            sim.enqueue_step()
        e1.record()
        torch.cuda.synchronize()
        sim.check_status()
        print(f"{a.config} graphs={graphs}: {e0.elapsed_time(e1) / a.steps:.4f} ms/step (device)",
              flush=True)


if __name__ == "__main__":
    main()
