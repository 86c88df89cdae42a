"""Helpers for the GPU-vs-oracle parity tests."""

from __future__ import annotations

import numpy as np

from golden_util import oracle_params, rel_l2

FIELDS9 = ("Ex", "Ey", "Ez", "Bx", "By", "Bz", "Jx", "Jy", "Jz")
PK = ("cx", "cy", "cz", "ox", "oy", "oz", "ux", "uy", "uz", "w")

# SURVEY.md §8c tolerances (10-100x the reference's own Serial-vs-BlockPool spread)
TOL_1STEP = {np.dtype(np.float64): 1e-13, np.dtype(np.float32): 1e-6}
TOL_FREE = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-4}
TOL_RESID = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-6}
TOL_GAUSS = {np.dtype(np.float64): 1e-13, np.dtype(np.float32): 1e-6}


def gpu_params(op, shape="tsc"):
    """Build the drop-in's SimParams from an oracle/golden params object."""
    from paper_1606_02862_b200.pic import SimParams, Species
    return SimParams(cells=op.cells, dx=op.dx, dy=op.dy, dz=op.dz, dt=op.dt,
                     species=tuple(Species(s.name, s.charge, s.mass, s.weight)
                                   for s in op.species),
                     particles_per_cell=op.particles_per_cell, super_cell=op.super_cell,
                     dtype=op.dtype, stream_velocity=op.stream_velocity,
                     perturbation=op.perturbation, thermal_u=op.thermal_u, shape=shape)


def sorted_records(pk: dict) -> dict:
    """Order-independent canonical form: lexsort on (cell, bit patterns)."""
    keys = []
    for k in reversed(PK):
        a = np.asarray(pk[k])
        if a.dtype.kind == "f":
            a = a.view(np.uint64 if a.dtype.itemsize == 8 else np.uint32)
        keys.append(a)
    order = np.lexsort(keys)
    return {k: np.asarray(pk[k])[order] for k in PK}


def assert_particles_bitwise(gpu_store, oracle_store):
    a = sorted_records(gpu_store.packed())
    b = sorted_records(oracle_store.packed())
    assert a["cx"].shape == b["cx"].shape, "census differs"
    for k in PK:
        bad = np.count_nonzero(a[k].view(np.uint8).reshape(a[k].shape[0], -1)
                               != b[k].view(np.uint8).reshape(b[k].shape[0], -1))
        assert bad == 0, f"{k}: {bad} records differ"
    np.testing.assert_array_equal(gpu_store.super_cell_counts(), oracle_store.super_cell_counts())


def occupancy(pk, cells):
    h = np.zeros(cells, dtype=np.int64)
    np.add.at(h, (pk["cx"], pk["cy"], pk["cz"]), 1)
    return h


def field_errors(gpu_fields, ref_fields_getter):
    """Relative L2 per lattice; ref_fields_getter(name) -> numpy (nx, ny, nz)."""
    return {n: rel_l2(gpu_fields.numpy(n), ref_fields_getter(n)) for n in FIELDS9}


def make_pair(meta, shape="tsc", validate=True):
    from oracle.pic import oracle_init_khi
    from paper_1606_02862_b200.pic import init_khi
    op = oracle_params(meta)
    order = {"cic": 1, "tsc": 2, "pcs": 3}[shape]
    seed = meta["config"]["seed"]
    gpu = init_khi(gpu_params(op, shape), seed=seed, validate=validate)
    orc = oracle_init_khi(op, seed=seed, validate=validate, shape_order=order, threads=8)
    return gpu, orc


def shadow_error(orc, steps=1):
    """Intrinsic rounding error of the storage-precision reference for the
    current state: relative L2 between the oracle stepped in its own dtype and
    a float64 shadow stepped from the same (exactly widened) state.  Used to
    state the field tolerance for f32 cases whose J is a cancellation of
    species currents (e.g. KHI pairs), where the reference itself is only
    accurate to ~1e-5.  Does not advance `orc`."""
    import copy
    from oracle.pic import OracleSim
    if orc.dtype == np.float64:
        return {n: 0.0 for n in FIELDS9}
    p32 = orc.params
    a = OracleSim(p32, validate=False, shape_order=orc.shape_order)
    import dataclasses
    if dataclasses.is_dataclass(p32):   # SimParams is frozen
        p64 = dataclasses.replace(p32, dtype=np.dtype(np.float64))
    else:
        p64 = copy.copy(p32)
        p64.dtype = np.dtype(np.float64)
    b = OracleSim(p64, validate=False, shape_order=orc.shape_order)
    for so, sa, sb in zip(orc.stores, a.stores, b.stores):
        pk = so.packed()
        scx, scy, scz = so.super_cell
        gx, gy, _ = so.sc_grid
        sc = (pk["cx"] // scx) + gx * ((pk["cy"] // scy) + gy * (pk["cz"] // scz))
        sa.load_packed(sc, pk)
        sb.load_packed(sc, {k: (v.astype(np.float64) if v.dtype.kind == "f" else v)
                            for k, v in pk.items()})
    for n in FIELDS9:
        setattr(a.fields, n, getattr(orc.fields, n).copy())
        setattr(b.fields, n, getattr(orc.fields, n).astype(np.float64))
    a.run(steps)
    b.run(steps)
    return {n: rel_l2(getattr(a.fields, n), getattr(b.fields, n)) for n in FIELDS9}


def field_tol(base, shadow, n):
    """Tolerance for lattice n: the stated bar, or 3x the reference's own
    intrinsic error when that is larger (ill-conditioned J)."""
    return max(base, 3.0 * shadow.get(n, 0.0))
