"""Generate golden fixtures from the UNMODIFIED reference (kernelweave.pic).

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Each case runs the reference's Serial back-end (deterministic accumulation
order, SPEC.md "Deposition determinism") from ``init_khi`` and dumps, at the
listed steps: all nine field lattices, the validation charge density, the
continuity residual, the diagnostics dict, and per species the canonical
``packed()`` arrays as SHA-256 digests plus per-super-cell counts and the
per-cell occupancy histogram.  The last step of each case also stores the
full packed arrays so mismatches can be localised.

The fixtures pin the CPU oracle (oracle/pic.py) bitwise and the CUDA path
within the SURVEY.md §8c tolerances.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = os.environ.get("KW_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from kernelweave.backends import SerialBackend  # noqa: E402
from kernelweave.pic.params import SimParams, Species, default_species  # noqa: E402
from kernelweave.pic.sim import init_khi  # noqa: E402
from kernelweave.pic import fields as kwf  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # C1 shape scaled down: thermal electrons, fp64 (reference default) and fp32
    "thermal_e_f64": dict(cells=(16, 8, 8), ppc=8, species="e", dtype="float64",
                          stream_velocity=0.0, perturbation=0.0, thermal_u=0.05,
                          seed=1, steps=(0, 1, 2, 6)),
    "thermal_e_f32": dict(cells=(16, 8, 8), ppc=8, species="e", dtype="float32",
                          stream_velocity=0.0, perturbation=0.0, thermal_u=0.05,
                          seed=1, steps=(0, 1, 2, 6)),
    # C3 shape scaled down: KHI + thermal noise, two species (mass ratio 1)
    "khi_pair_f32": dict(cells=(16, 16, 4), ppc=4, species="pair", mass_ratio=1.0,
                         dtype="float32", stream_velocity=0.2, perturbation=0.01,
                         thermal_u=0.01, seed=3, steps=(0, 1, 4)),
    # C2 shape scaled down: e/ion 1836, hot enough to cross super cells often
    "eion_f32": dict(cells=(8, 16, 8), ppc=2, species="pair", mass_ratio=1836.0,
                     dtype="float32", stream_velocity=0.0, perturbation=0.0,
                     thermal_u=0.3, seed=2, steps=(0, 1, 3)),
    # anisotropic cell sizes, fp64, non-default super cell
    "aniso_f64": dict(cells=(8, 8, 8), ppc=2, species="pair", mass_ratio=4.0,
                      dtype="float64", stream_velocity=0.3, perturbation=0.05,
                      thermal_u=0.1, seed=7, steps=(0, 1, 3), deltas=(0.7, 1.0, 1.3),
                      super_cell=(4, 4, 4)),
}


# BASELINE-scale cases (SURVEY.md §8c golden plan): C1 in full (32^3, 8 ppc,
# electrons, thermal 0.05, TSC, 100 steps) in fp64 and fp32, and 32^3
# proxies of C2-C4 with their ppc, species and distribution (10 steps).
# Stored as SHA-256 digests of every lattice and every packed particle array
# at each dumped step (they pin the oracle bitwise at scale,
# tests/test_oracle_golden.py), per-cell occupancy and per-super-cell counts
# at each dump, diagnostics, and -- for C1 -- the nine lattices at the last
# step (the GPU free-running test compares against the reference's own).
BIG = {
    "c1_tsc_f64": dict(cells=(32, 32, 32), ppc=8, species="e", dtype="float64",
                       stream_velocity=0.0, perturbation=0.0, thermal_u=0.05,
                       seed=1, steps=(0, 1, 10, 100), fields_at=(100,)),
    "c1_tsc_f32": dict(cells=(32, 32, 32), ppc=8, species="e", dtype="float32",
                       stream_velocity=0.0, perturbation=0.0, thermal_u=0.05,
                       seed=1, steps=(0, 1, 10, 100), fields_at=(100,)),
    "c2p_f32": dict(cells=(32, 32, 32), ppc=25, species="pair", mass_ratio=1836.0,
                    dtype="float32", stream_velocity=0.0, perturbation=0.0, thermal_u=0.05,
                    seed=2, steps=(0, 1, 10), fields_at=()),
    "c3p_f32": dict(cells=(32, 32, 32), ppc=16, species="pair", mass_ratio=1.0,
                    dtype="float32", stream_velocity=0.2, perturbation=0.01, thermal_u=0.01,
                    seed=3, steps=(0, 1, 10), fields_at=()),
    "c4p_f32": dict(cells=(32, 32, 32), ppc=32, species="e", dtype="float32",
                    stream_velocity=0.0, perturbation=0.0, thermal_u=0.05,
                    seed=4, steps=(0, 1, 10), fields_at=()),
}


def run_big(name, c):
    import time
    params = make_params(c)
    t0 = time.time()
    sim = init_khi(params, seed=c["seed"], backend=SerialBackend(), validate=True)
    out = {}
    meta = {"case": name, "config": {k: v for k, v in c.items() if k != "fields_at"},
            "dt": params.dt, "steps": {}, "digests": True}
    last = max(c["steps"])
    for t in range(last + 1):
        if t in c["steps"]:
            key = f"t{t}"
            f = sim.fields
            sm = {"residual": sim.last_residual, "diagnostics": sim.diagnostics(),
                  "census": sim.census(), "species": [],
                  "fields": {n: digest(getattr(f, n)) for n in kwf.ALL_COMPONENTS}}
            for i, st in enumerate(sim.stores):
                pk = st.packed()
                sm["species"].append({k: digest(v) for k, v in pk.items()})
                out[f"{key}_s{i}_sc_counts"] = sc_counts(st)
                out[f"{key}_s{i}_occupancy"] = occupancy(st, params.cells.as_tuple()).astype(np.int16)
            if t in c["fields_at"]:
                for n in kwf.ALL_COMPONENTS:
                    out[f"{key}_{n}"] = getattr(f, n).copy()
            meta["steps"][key] = sm
        if t < last:
            sim.step()
    meta["reference_seconds"] = time.time() - t0
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    with open(os.path.join(OUT, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(name, "census", sim.census(), "residual", sim.last_residual,
          f"{meta['reference_seconds']:.1f} s", flush=True)


def make_params(c):
    if c["species"] == "e":
        sp = (Species("electron", -1.0, 1.0, 1.0 / c["ppc"]),)
    else:
        sp = default_species(c["ppc"], c.get("mass_ratio", 1.0))
    dx, dy, dz = c.get("deltas", (1.0, 1.0, 1.0))
    return SimParams(cells=c["cells"], dx=dx, dy=dy, dz=dz, species=sp,
                     particles_per_cell=c["ppc"],
                     super_cell=c.get("super_cell", (8, 8, 4)),
                     dtype=np.dtype(c["dtype"]),
                     stream_velocity=c["stream_velocity"],
                     perturbation=c["perturbation"], thermal_u=c["thermal_u"])


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def occupancy(store, cells):
    pk = store.packed(("cx", "cy", "cz"))
    h = np.zeros(cells, dtype=np.int32)
    np.add.at(h, (pk["cx"], pk["cy"], pk["cz"]), 1)
    return h


def sc_counts(store):
    cnt = np.zeros(store.n_super_cells, dtype=np.int32)
    for sc in range(store.n_super_cells):
        cnt[sc] = sum(int(store.nfilled[f]) for f in store.frames_of(sc))
    return cnt


def run_case(name, c):
    params = make_params(c)
    sim = init_khi(params, seed=c["seed"], backend=SerialBackend(), validate=True)
    out = {}
    meta = {"case": name, "config": c, "dt": params.dt, "steps": {}}
    last = max(c["steps"])
    for t in range(last + 1):
        if t in c["steps"]:
            key = f"t{t}"
            f = sim.fields
            for n in kwf.ALL_COMPONENTS:
                out[f"{key}_{n}"] = getattr(f, n).copy()
            out[f"{key}_rho"] = sim.charge_density()
            sm = {"residual": sim.last_residual, "diagnostics": sim.diagnostics(),
                  "census": sim.census(), "species": []}
            for i, st in enumerate(sim.stores):
                pk = st.packed()
                sm["species"].append({k: digest(v) for k, v in pk.items()})
                out[f"{key}_s{i}_sc_counts"] = sc_counts(st)
                out[f"{key}_s{i}_occupancy"] = occupancy(st, params.cells.as_tuple()).astype(np.int16)
                if t == last or t == 0:
                    for k, v in pk.items():
                        out[f"{key}_s{i}_{k}"] = v
            meta["steps"][key] = sm
        if t < last:
            sim.step()
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    with open(os.path.join(OUT, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(name, "census", sim.census(), "residual", sim.last_residual)


def kat():
    """SPEC.md known-answer values computed by the reference functions."""
    from kernelweave.pic.pusher import boris_push
    from kernelweave.pic.deposit import _shape5
    rng = np.random.default_rng(123)
    xs = rng.uniform(-0.99, 1.99, 64)
    res = {
        "tsc_half": list(kwf.tsc_weights(0.5)),
        "shape5_x": xs.tolist(),
        "shape5": [list(map(float, _shape5(float(x)))) for x in xs],
        "boris_b0": list(boris_push((0.1, -0.2, 0.3), (0.5, 0.0, 0.0), (0.0, 0.0, 0.0),
                                    -1.0, 1.0, 0.5)),
    }
    with open(os.path.join(OUT, "kat.json"), "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES) + list(BIG)
    for n in names:
        if n in BIG:
            run_big(n, BIG[n])
        else:
            run_case(n, CASES[n])
    if not sys.argv[1:]:
        kat()
