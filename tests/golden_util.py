"""Shared helpers to load the golden fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import hashlib
import json
import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ("thermal_e_f64", "thermal_e_f32", "khi_pair_f32", "eion_f32", "aniso_f64")


def load_case(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        meta = json.load(fh)
    data = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return meta, data


def species_of(c):
    S = SimpleNamespace
    if c["species"] == "e":
        return (S(name="electron", charge=-1.0, mass=1.0, weight=1.0 / c["ppc"]),)
    w = 1.0 / c["ppc"]
    return (S(name="electron", charge=-1.0, mass=1.0, weight=w),
            S(name="ion", charge=1.0, mass=float(c.get("mass_ratio", 1.0)), weight=w))


def oracle_params(meta):
    """Duck-typed params object accepted by oracle.pic (mirrors SimParams)."""
    c = meta["config"]
    dx, dy, dz = c.get("deltas", (1.0, 1.0, 1.0))
    return SimpleNamespace(
        cells=tuple(c["cells"]), dx=dx, dy=dy, dz=dz, dt=meta["dt"],
        species=species_of(c), particles_per_cell=c["ppc"],
        super_cell=tuple(c.get("super_cell", (8, 8, 4))), dtype=np.dtype(c["dtype"]),
        stream_velocity=c["stream_velocity"], perturbation=c["perturbation"],
        thermal_u=c["thermal_u"])


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    d = np.linalg.norm(a - b)
    return float(d / nb) if nb > 0 else float(d)


# BASELINE-scale cases (tests/golden/make_golden.py BIG): digests at every
# dumped step, occupancy and super-cell counts, C1 lattices at t = 100.
BIG_CASES = ("c1_tsc_f64", "c1_tsc_f32", "c2p_f32", "c3p_f32", "c4p_f32")
