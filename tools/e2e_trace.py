"""Per-step wall time of the e2e leg of bench.py (load_state from pinned host
buffers, then Simulation.step() K times), to see where e2e loses against
the device-timed value.

    python tools/e2e_trace.py [--config c2] [--steps 100]
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    import torch
    import bench
    from paper_1606_02862_b200.pic import init_khi
    p, seed = bench.make_params(a.config)
    sim = init_khi(p, seed=seed, validate=False, rng="device")
    for _ in range(a.steps + 3):
        sim.enqueue_step()
    sim.check_status()
    names = ("Ex", "Ey", "Ez", "Bx", "By", "Bz", "Jx", "Jy", "Jz")
    host_fields = {n: sim.fields.numpy(n) for n in names}
    host_parts = [{k: v.cpu().pin_memory() for k, v in st.packed_device().items()}
                  for st in sim.stores]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim.load_state(fields=host_fields, particles=host_parts)
    torch.cuda.synchronize()
    print(f"load_state {1e3 * (time.perf_counter() - t0):.1f} ms; frames "
          f"{[st.frames_per_sc for st in sim.stores]}", flush=True)
    times = []
    for i in range(a.steps):
        t0 = time.perf_counter()
        sim.step()
        torch.cuda.synchronize()
        times.append(1e3 * (time.perf_counter() - t0))
    times_s = sorted(times)
    print(f"step(): mean {sum(times) / len(times):.3f} median {times_s[len(times) // 2]:.3f} "
          f"max {times_s[-1]:.3f} ms; frames {[st.frames_per_sc for st in sim.stores]}")
    print("slowest:", sorted(range(len(times)), key=lambda i: -times[i])[:5],
          [round(t, 1) for t in sorted(times, reverse=True)[:5]])


if __name__ == "__main__":
    main()
