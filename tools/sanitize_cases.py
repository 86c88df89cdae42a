"""Small CUDA workloads for compute-sanitizer (racecheck / synccheck /
memcheck / initcheck), covering every kernel of the library: one-step
advance + shift + Yee + validation for CIC/TSC/PCS in float32 and float64,
a dense hot plasma (mid-loop queue drains, PCS ring wrap-around), a
non-default super cell, the fused z-slab loopback (plane-table J flush,
guard extract / load_counted, plane pulls), store load/export/repack,
gather_fields and the device init.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1606_02862_b200.pic import (MacroParticle, SimParams, Species, default_species,  # noqa: E402
                                       gather_fields, init_khi)
from paper_1606_02862_b200.pic.decomp import DecomposedSimulation, LoopbackTransport  # noqa: E402


def case(name, fn):
    fn()
    torch.cuda.synchronize()
    print("case ok:", name, flush=True)


def one_step(shape, dtype, sc=(8, 8, 4), ppc=4, thermal=0.3, cells=(16, 16, 8)):
    def run():
        p = SimParams(cells=cells, species=default_species(ppc, 4.0), particles_per_cell=ppc,
                      dtype=dtype, thermal_u=thermal, stream_velocity=0.1, perturbation=0.01,
                      shape=shape, super_cell=sc)
        sim = init_khi(p, seed=3, validate=True)
        sim.step()
        sim.step()
        sim.diagnostics()
        e, b = gather_fields(sim.fields, [MacroParticle((1, 2, 3), (0.5, 0.25, 1.0), (0, 0, 0))])
        pk = sim.stores[0].packed()
        assert len(pk["cx"]) > 0
    return run


def dense(shape):
    def run():
        p = SimParams(cells=(16, 16, 8), species=default_species(40, 1836.0),
                      particles_per_cell=40, dtype=np.float32, thermal_u=0.3, shape=shape)
        sim = init_khi(p, seed=21, validate=False)
        sim.step()
    return run


def zslab(fuse):
    def run():
        p = SimParams(cells=(16, 16, 24), species=default_species(4, 4.0), particles_per_cell=4,
                      dtype=np.float32, stream_velocity=0.2, perturbation=0.05, thermal_u=0.1)
        ref = init_khi(p, seed=9, validate=False)
        dec = DecomposedSimulation(p, 2, range(2), LoopbackTransport(), fuse_j=fuse)
        dec.load_global(particles=[st.packed() for st in ref.stores])
        dec.refresh_guards()
        dec.step()
        dec.step()
        dec.census()
    return run


def device_init():
    p = SimParams(cells=(16, 16, 8), species=default_species(4, 1836.0), particles_per_cell=4,
                  dtype=np.float32, thermal_u=0.05)
    sim = init_khi(p, seed=2, validate=False, rng="device")
    sim.step()


if __name__ == "__main__":
    which = sys.argv[1:] or ["all"]
    cases = []
    for dt in (np.float32, np.float64):
        for sh in ("cic", "tsc", "pcs"):
            cases.append((f"one_step_{sh}_{np.dtype(dt).name}", one_step(sh, dt)))
    cases.append(("one_step_tsc_f32_sc444", one_step("tsc", np.float32, sc=(4, 4, 4))))
    for sh in ("tsc", "pcs"):
        cases.append((f"dense_{sh}", dense(sh)))
    cases.append(("zslab_fused", zslab(True)))
    cases.append(("zslab_messages", zslab(False)))
    cases.append(("device_init", device_init))
    for name, fn in cases:
        if "all" in which or name in which:
            case(name, fn)
