"""CPU-side checks of the boundary and the host logic (no GPU needed).

* libkwb200.so loads and exports every entry point include/kwb200.h
  declares (no compute calls here);
* SimParams validation mirrors the reference (ValueError on CFL and
  divisibility);
* the host-side init_khi generator reproduces the reference's initial state
  bitwise (golden t0 digests) -- this is the exact data the device store is
  loaded with.
"""

import ctypes
import os
import re

import numpy as np
import pytest

from golden_util import CASES, digest, load_case, oracle_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "kwb200.h")) as fh:
        src = fh.read()
    return sorted(set(re.findall(r"\b(kwb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_1606_02862_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.kwb_version() == 1


def test_library_rejects_bad_arguments_without_gpu():
    """Argument validation happens before any CUDA call."""
    from paper_1606_02862_b200 import _lib
    lib = _lib.load()
    g = _lib.Grid(nx=16, ny=16, nz=8, scx=8, scy=8, scz=3, gx=2, gy=2, gz=2, dtype=0,
                  dx=1.0, dy=1.0, dz=1.0, dt=0.5)
    rc = lib.kwb_particles_shift(ctypes.byref(g), None, None, None, None)
    assert rc == -1
    assert b"does not tile" in lib.kwb_last_error()
    rc = lib.kwb_fields_faraday_half(None, _lib.Ptr3(), _lib.Ptr3(), 0.5, None)
    assert rc == -1


def test_species_entry_points_reject_bad_arguments_without_gpu():
    """kwb_particles_advance_species / _split validate the species count,
    the shape order and every store (workspace included) before any launch
    (fake device pointers: nothing may reach the GPU)."""
    from paper_1606_02862_b200 import _lib
    lib = _lib.load()
    g = _lib.Grid(nx=16, ny=16, nz=8, scx=8, scy=8, scz=4, gx=2, gy=2, gz=2, dtype=0,
                  dx=1.0, dy=1.0, dz=1.0, dt=0.5)
    fake = 0x10000

    def store(frames):
        st = _lib.StoreC()
        for c in ("ox", "oy", "oz", "ux", "uy", "uz", "w", "front", "back"):
            setattr(st, c, fake)
        st.frames_per_sc = frames
        return st
    ex = _lib.ExchangeC()
    for c in ("ox", "oy", "oz", "ux", "uy", "uz", "w", "cx", "cy", "cz", "dest", "count"):
        setattr(ex, c, fake)
    ex.capacity = 16
    sp = (_lib.SpeciesC * 5)()
    ins = (_lib.StoreC * 5)(*[store(8) for _ in range(5)])
    outs = (_lib.StoreC * 5)(*[store(8) for _ in range(5)])
    ptr = _lib.Ptr3(fake, fake, fake)
    status = fake
    call = lambda name, *a: getattr(lib, name)(ctypes.byref(g), *a)
    # five species: more than kMaxSpecies
    rc = call("kwb_particles_advance_species", 5, sp, ins, outs, ctypes.byref(ex), ptr, ptr, ptr,
              None, 2, status, None)
    assert rc == -1 and b"at most" in lib.kwb_last_error()
    # split: a workspace store of another frame count
    wss = (_lib.StoreC * 2)(store(8), store(9))
    rc = call("kwb_particles_advance_split", 2, sp, ins, outs, wss, ctypes.byref(ex), ptr, ptr,
              ptr, None, 2, status, None)
    assert rc == -1 and b"frames_per_sc" in lib.kwb_last_error()
    # split: an incomplete workspace store
    bad = store(8)
    bad.w = None
    wss = (_lib.StoreC * 2)(store(8), bad)
    rc = call("kwb_particles_advance_split", 2, sp, ins, outs, wss, ctypes.byref(ex), ptr, ptr,
              ptr, None, 1, status, None)
    assert rc == -1 and b"workspace" in lib.kwb_last_error()
    # split: unknown shape order
    wss = (_lib.StoreC * 2)(store(8), store(8))
    rc = call("kwb_particles_advance_split", 2, sp, ins, outs, wss, ctypes.byref(ex), ptr, ptr,
              ptr, None, 5, status, None)
    assert rc == -1 and b"shape_order" in lib.kwb_last_error()


def test_simparams_validation():
    from paper_1606_02862_b200.pic import SimParams, default_species
    with pytest.raises(ValueError):
        SimParams(cells=(16, 16, 6))               # (8,8,4) does not divide
    with pytest.raises(ValueError):
        SimParams(cells=(16, 16, 8), dt=1.0)        # CFL
    with pytest.raises(ValueError):
        SimParams(cells=(16, 16, 8), shape="ngp")
    p = SimParams(cells=(16, 16, 8))
    assert p.dt == pytest.approx(0.95 / np.sqrt(3.0))
    assert p.species == default_species(16)
    assert p.frame_capacity == 256 and p.shape_order == 2


def test_cpu_backend_is_rejected():
    from paper_1606_02862_b200.errors import CapabilityError
    from paper_1606_02862_b200.pic import SimParams, Simulation

    class SerialBackend:  # a reference-style CPU back-end
        kind = "serial"

    with pytest.raises(CapabilityError):
        Simulation(SimParams(cells=(16, 16, 8)), backend=SerialBackend())


@pytest.mark.parametrize("name", CASES)
def test_host_init_matches_reference(name):
    from paper_1606_02862_b200.pic import SimParams, Species
    from paper_1606_02862_b200.pic.sim import khi_species_particles
    meta, data = load_case(name)
    op = oracle_params(meta)
    p = SimParams(cells=op.cells, dx=op.dx, dy=op.dy, dz=op.dz, dt=op.dt,
                  species=tuple(Species(s.name, s.charge, s.mass, s.weight) for s in op.species),
                  particles_per_cell=op.particles_per_cell, super_cell=op.super_cell,
                  dtype=op.dtype, stream_velocity=op.stream_velocity,
                  perturbation=op.perturbation, thermal_u=op.thermal_u)
    t0 = meta["steps"]["t0"]["species"]
    for i, sp in enumerate(p.species):
        rng = np.random.default_rng((meta["config"]["seed"], i)) if p.thermal_u > 0 else None
        n_sc = p.super_cell_grid.volume
        parts = [khi_species_particles(p, meta["config"]["seed"], i, b, min(n_sc, b + 3), rng)
                 for b in range(0, n_sc, 3)]   # chunked: the stream must continue
        a = {k: np.concatenate([q[k] for q in parts]) for k in parts[0]}
        for k in ("cx", "cy", "cz"):
            assert digest(a[k].astype(np.int32)) == t0[i][k], k
        for k in ("ox", "oy", "oz", "ux", "uy", "uz"):
            assert digest(a[k].astype(p.dtype)) == t0[i][k], k
        assert digest(np.full(a["cx"].shape, sp.weight, dtype=p.dtype)) == t0[i]["w"]
