"""Where the e2e leg of bench.py spends its wall time: host<->device copy
bandwidth of plain pinned buffers (the PCIe ceiling), then load_state
(copies + column build), the steps, and packed(out=...) (export kernel +
copies), each timed separately with synchronisation.

    python tools/e2e_breakdown.py [--config c2] [--steps 20]
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

    def wall(fn, reps=3):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    nbytes = 1 << 30
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    t = wall(lambda: d.copy_(h, non_blocking=True))
    print(f"pinned H2D 1 GiB: {nbytes / t / 1e9:6.1f} GB/s")
    t = wall(lambda: h.copy_(d, non_blocking=True))
    print(f"pinned D2H 1 GiB: {nbytes / t / 1e9:6.1f} GB/s")
    s2 = torch.cuda.Stream()

    def both():
        d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s2)
    t = wall(both)
    print(f"pinned H2D + D2H concurrently: {2 * nbytes / t / 1e9:6.1f} GB/s total")
    chunks = [(h[i:i + nbytes // 8], d[i:i + nbytes // 8]) for i in range(0, nbytes, nbytes // 8)]
    t = wall(lambda: [dd.copy_(hh, non_blocking=True) for hh, dd in chunks])
    print(f"pinned H2D 8 x 128 MiB: {nbytes / t / 1e9:6.1f} GB/s")
    del h, d, h2, d2, chunks

    p, seed = bench.make_params(a.config)
    sim = init_khi(p, seed=seed, validate=False, rng="device")
    for _ in range(3):
        sim.step()
    names = ("Ex", "Ey", "Ez", "Bx", "By", "Bz", "Jx", "Jy", "Jz")
    host_fields = {n: torch.from_numpy(sim.fields.numpy(n)).pin_memory() for n in names}
    host_parts = [{k: v.cpu().pin_memory() for k, v in st.packed_device().items()}
                  for st in sim.stores]
    h2d = sum(v.numel() * v.element_size() for dd in host_parts for v in dd.values())
    host_out = [{k: torch.empty(int(v.numel() * 1.05) + 1024, dtype=v.dtype).pin_memory()
                 for k, v in dd.items()} for dd in host_parts]

    t = wall(lambda: sim.load_state(fields=host_fields, particles=host_parts))
    print(f"load_state: {t * 1e3:7.1f} ms ({h2d / t / 1e9:5.1f} GB/s of particle records)")
    t = wall(lambda: sim.load_state(fields=host_fields))
    print(f"  fields only: {t * 1e3:7.1f} ms")
    for i, st in enumerate(sim.stores):
        t = wall(lambda: st.load_packed(host_parts[i]))
        print(f"  species {i} load_packed: {t * 1e3:7.1f} ms")
    sim.load_state(fields=host_fields, particles=host_parts)
    t = wall(lambda: [sim.step() for _ in range(a.steps)], reps=1)
    print(f"{a.steps} x step(): {t * 1e3:7.1f} ms ({t / a.steps * 1e3:.2f} ms/step)")
    t = wall(lambda: [st.packed_device() for st in sim.stores])
    print(f"export kernels (packed_device, both species): {t * 1e3:7.1f} ms")
    t = wall(lambda: [st.packed(out=buf) for st, buf in zip(sim.stores, host_out)])
    print(f"packed(out=pinned), both species: {t * 1e3:7.1f} ms ({h2d / t / 1e9:5.1f} GB/s)")


if __name__ == "__main__":
    main()
