"""The PIC cycle on B200 (API of kernelweave.pic.sim, reference
pic/sim.py:33-328).

``Simulation.step()`` runs, on one CUDA stream and with no host round trip
inside the cycle:

    J = 0
    per species:  kwb_particles_advance  (gather -> push -> move -> deposit,
                                          compaction into the spare columns)
                  kwb_particles_shift    (leavers into their new super cell)
    kwb_fields_faraday_half -> kwb_fields_ampere -> kwb_fields_faraday_half
    [validate]    kwb_charge_density + kwb_continuity_residual (+ Gauss drift)

then reads one small status word block (move violations, capacity) and
raises ``ContractViolation`` exactly where the reference's DepositKernel
would (pic/kernels.py:405-408).  The reference's order -- all species
deposit, then migrate, then the field update -- is preserved.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch

from .. import _lib
from ..backend import B200Backend
from ..errors import AllocationError, CapabilityError, ContractViolation
from ..workdiv import make_work_division
from .fields import ALL_COMPONENTS, YeeFieldSet, div_b, div_j, field_energy  # noqa: F401
from .params import SimParams, default_species  # noqa: F401
from .particles import SuperCellStore

STRATEGIES = ("elements", "threads")
EXCHANGE_FRACTION = 0.25


def _near_cubic_factors(n: int) -> tuple[int, int, int]:
    """Deterministic balanced factorisation (pic/sim.py:36-52)."""
    best, best_score = (n, 1, 1), n
    for px in range(1, n + 1):
        if n % px:
            continue
        rest = n // px
        for py in range(1, rest + 1):
            if rest % py:
                continue
            pz = rest // py
            score = max(px, py, pz) - min(px, py, pz)
            if score < best_score:
                best_score, best = score, (px, py, pz)
    return best


class _nvtx:
    """NVTX range around one stage of the cycle (visible in nsys / ncu
    --nvtx): advance, shift, fields, validate.  Host-side only; a range
    inside a CUDA-graph capture costs nothing at replay."""

    __slots__ = ("name",)

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        torch.cuda.nvtx.range_push(self.name)

    def __exit__(self, *exc):
        torch.cuda.nvtx.range_pop()
        return False


def _grid_struct(p: SimParams) -> _lib.Grid:
    g = _lib.Grid()
    g.nx, g.ny, g.nz = p.cells.as_tuple()
    g.scx, g.scy, g.scz = p.super_cell.as_tuple()
    g.gx, g.gy, g.gz = p.super_cell_grid.as_tuple()
    g.dtype = _lib.KWB_F32 if p.dtype == np.float32 else _lib.KWB_F64
    g.dx, g.dy, g.dz, g.dt = p.dx, p.dy, p.dz, p.dt
    return g


def _species_struct(p: SimParams, s) -> _lib.SpeciesC:
    c = _lib.SpeciesC()
    deltas = (p.dx, p.dy, p.dz)
    vol = p.cell_volume
    c.qm_half_dt = s.charge * p.dt / (2.0 * s.mass)            # pic/sim.py:101-103
    for a in range(3):
        c.fac[a] = -s.charge * deltas[a] / (p.dt * vol)       # pic/sim.py:104-110
        c.dt_d[a] = p.dt / deltas[a]                           # pic/sim.py:100
    c.q_inv_vol = s.charge / vol                               # pic/sim.py:188
    c.charge, c.mass = s.charge, s.mass
    return c


class _Exchange:
    """Leaver buffer shared by the species of one Simulation."""

    def __init__(self, capacity, tdtype, device):
        self.capacity = int(capacity)
        for c in ("ox", "oy", "oz", "ux", "uy", "uz", "w"):
            setattr(self, c, torch.empty(self.capacity, dtype=tdtype, device=device))
        for c in ("cx", "cy", "cz", "dest"):
            setattr(self, c, torch.empty(self.capacity, dtype=torch.int32, device=device))
        self.count = torch.zeros(1, dtype=torch.int32, device=device)
        e = _lib.ExchangeC()
        for c in ("ox", "oy", "oz", "ux", "uy", "uz", "w", "cx", "cy", "cz", "dest", "count"):
            setattr(e, c, getattr(self, c).data_ptr())
        e.capacity = self.capacity
        self.cstruct = e


class Simulation:
    """Fields + per-species super-cell stores, stepped on one B200."""

    def __init__(self, params: SimParams, backend=None, strategy="elements", validate=True):
        if strategy not in STRATEGIES:
            raise ValueError(f"strategy must be one of {STRATEGIES}")
        if backend is None:
            backend = B200Backend()
        if not isinstance(backend, B200Backend):
            raise CapabilityError(
                f"{type(backend).__name__} is not supported: this build runs the PIC cycle "
                "on a B200 only (no CPU back-end, no fallback)")
        _lib.load()
        self.params = params
        self.backend = backend
        self.device = backend.device
        self.strategy = strategy
        self.validate = validate
        self.step_count = 0
        p = params
        self.shape_order = p.shape_order
        self.fields = YeeFieldSet(p.cells, p.dx, p.dy, p.dz, p.dtype, self.device)
        self.stores = [SuperCellStore(p.cells, p.super_cell, p.dtype, self.device)
                       for _ in p.species]
        grid = p.super_cell_grid
        n_sc = grid.volume
        sc = p.super_cell.as_tuple()
        s = np.arange(n_sc)
        self.origins = np.stack([(s % grid.x) * sc[0], ((s // grid.x) % grid.y) * sc[1],
                                 (s // (grid.x * grid.y)) * sc[2]], axis=1).astype(np.int64)
        hw = 3 if self.shape_order == 3 else 2
        cells = p.cells.as_tuple()
        # wrapped deposit-tile -> grid maps (pic/sim.py:88-94; halo 3 for PCS)
        self.maps = tuple(((self.origins[:, a:a + 1] - hw + np.arange(sc[a] + 2 * hw)[None, :])
                           % cells[a]).astype(np.int64) for a in range(3))
        self.tile_shape = tuple(sc[a] + 2 * hw for a in range(3))
        self._grid = _grid_struct(p)
        self._species = [_species_struct(p, sp) for sp in p.species]
        # one particle-phase call for all species (two species: one fused
        # launch); False: the reference's per-species launches
        self.fuse_species = os.environ.get("KWB_PER_SPECIES", "0") != "1" and len(p.species) <= 4
        # advance as two kernels per species (dense push, then deposit/shift;
        # csrc/push.cuh) -- CIC/TSC only
        self.split_advance = (self.fuse_species and self.shape_order != 3 and
                              os.environ.get("KWB_SPLIT", "0") == "1")
        self._status = torch.zeros((len(p.species), _lib.STATUS_WORDS), dtype=torch.int32,
                                   device=self.device)
        self._status_host = torch.zeros_like(self._status, device="cpu").pin_memory()
        self._status_ring = [torch.zeros_like(self._status_host).pin_memory() for _ in range(2)]
        self._pending = []
        self._exchange = None
        # CUDA graphs of the whole cycle for enqueue_step (validate=False):
        # one per (current, spare) buffer assignment, re-captured whenever a
        # buffer is reallocated.  Launch-bound grids (C1: seven launches of
        # 10-70 us) run as one graph launch.
        self.use_graphs = os.environ.get("KWB_NO_GRAPHS", "") == ""
        self._graphs = {}
        self._rho_prev = None
        self._G_prev = None
        self._resid = torch.zeros(2, dtype=torch.float64, device=self.device)
        self._wd = None

    # -- launch plumbing ------------------------------------------------------
    def work_division(self):
        """Descriptive: one block per super cell (the CUDA mapping is fixed)."""
        if self._wd is None:
            grid, sc = self.params.super_cell_grid, self.params.super_cell
            if self.strategy == "elements":
                self._wd = make_work_division(grid, (1, 1, 1), sc)
            else:
                self._wd = make_work_division(grid, sc, (1, 1, 1))
        return self._wd

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def _E(self):
        return _lib.ptr3([self.fields.storage(n) for n in ("Ex", "Ey", "Ez")])

    def _B(self):
        return _lib.ptr3([self.fields.storage(n) for n in ("Bx", "By", "Bz")])

    def _J(self):
        return _lib.ptr3([self.fields.storage(n) for n in ("Jx", "Jy", "Jz")])

    def _exchange_buffer(self) -> _Exchange:
        # species-fused launches share the buffer between the species
        need = sum(st.loaded for st in self.stores)
        cap = int(math.ceil(EXCHANGE_FRACTION * need)) + 65536
        if self._exchange is None or self._exchange.capacity < min(cap, need + 65536):
            self._exchange = _Exchange(min(cap, need + 65536), self.stores[0].tdtype, self.device)
        return self._exchange

    # -- the PIC cycle ------------------------------------------------------
    def step(self):
        """One PIC cycle with the reference's synchronous semantics: raises
        ContractViolation before the field update if a particle moved a full
        cell (pic/kernels.py:405-408).  If a cell column or the exchange
        buffer ran full, the particle phase is undone (its input columns are
        intact -- the advance is double-buffered), capacity grows, and the
        phase is redone, so no particle is ever lost."""
        self._begin_step()
        for _attempt in range(6):
            self._enqueue_particles()
            st = self._read_status()
            lost = st[:, _lib.ST_EXCH_OVERFLOW].sum() + st[:, _lib.ST_STORE_OVERFLOW].sum()
            if int(lost) == 0:
                break
            self._undo_particles(st)
        else:
            raise AllocationError("particle phase keeps overflowing its capacity")
        moved = int(st[:, _lib.ST_MOVE_ERRORS].sum())
        if moved:
            raise ContractViolation(
                f"{moved} particle(s) moved a full cell or more before deposit")
        self._enqueue_fields()
        self.step_count += 1
        # the field update does not touch the status words: apply the ones
        # read above instead of a second synchronising read
        self._drain_status()
        self._apply_status(st)

    def enqueue_step(self):
        """Launch one full PIC cycle on the current stream without waiting for
        it (bench path).  The status words of every step are copied to pinned
        host memory behind an event and inspected two steps later (by then
        the event has long completed, so no stall): columns passing GROW_AT
        grow before they can overflow, and any violation raises at the latest
        in check_status().  With validate=False the cycle is replayed from a
        CUDA graph (captured on first use of each buffer assignment)."""
        self._drain_status(keep=1)
        if self.use_graphs and not self.validate and self.step_count > 0:
            self._graph_step()
        else:
            self._begin_step()
            self._enqueue_particles()
            self._enqueue_fields()
        self.step_count += 1
        self._post_status()

    def _graph_key(self):
        ex = self._exchange_buffer()
        key = [ex.count.data_ptr(), ex.capacity, self.fields._buf.data_ptr()]
        for st in self.stores:
            st.spare()   # both column buffers exist before a capture
            key += [st._cols[0].ox.data_ptr(), st._cols[1].ox.data_ptr(), st.frames_per_sc]
            if self.split_advance:
                key.append(st.workspace().ox.data_ptr())
        return tuple(key)

    def _graph_step(self):
        key = self._graph_key()
        g = self._graphs.get(key)
        if g is None:
            if len(self._graphs) >= 4:   # buffers were reallocated: drop stale graphs
                self._graphs.clear()
            cur = torch.cuda.current_stream(self.device)
            cap = torch.cuda.Stream(self.device)
            cap.wait_stream(cur)
            g = torch.cuda.CUDAGraph()
            # capture_begin/end directly: torch.cuda.graph() would also run
            # gc.collect() and empty the caching allocator (~0.2 s per capture)
            with torch.cuda.stream(cap):
                g.capture_begin()
                try:
                    self._enqueue_particles()
                    self._enqueue_fields()
                finally:
                    g.capture_end()
            cur.wait_stream(cap)
            for st in self.stores:   # the capture only recorded the work: undo its swaps
                st.swap()
            self._graphs[key] = g
        g.replay()
        for st in self.stores:
            st.swap()

    def _post_status(self):
        """Copy this step's status words to pinned memory behind an event."""
        slot = self._status_ring[self.step_count % 2]
        slot.copy_(self._status, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        self._pending.append((slot, ev))

    def _drain_status(self, keep=0):
        while len(self._pending) > keep:
            slot, ev = self._pending.pop(0)
            ev.synchronize()
            self._apply_status(slot.clone())

    def _begin_step(self):
        if self.validate and self._rho_prev is None:
            self._rho_prev = self._charge_density_storage()
            self._G_prev = torch.zeros_like(self._rho_prev)
            _lib.call("kwb_continuity_residual", ctypes.byref(self._grid),
                      self._rho_prev.data_ptr(), None, self._J(), self._E(),
                      self._G_prev.data_ptr(), self._resid.data_ptr(), self._stream())

    def _enqueue_particles(self, zero_j=True):
        """zero_j=False: J was zeroed by the caller (z-slab fused halo: other
        slabs' deposits land in this slab's J before its own advance)."""
        stream = self._stream()
        g = ctypes.byref(self._grid)
        E, B, J = self._E(), self._B(), self._J()
        _lib.call("kwb_zero_step", g, ctypes.cast(J, ctypes.c_void_p) if zero_j else None,
                  self._status.data_ptr(), self._status.numel(), stream)
        ex = self._exchange_buffer()
        jpl = getattr(self, "_jplanes", None)
        if self.fuse_species:
            # every species' advance + shift in one call: two species share
            # one fused launch (kwb_particles_advance_species)
            n = len(self.stores)
            ins = (_lib.StoreC * n)(*[st.current.cstruct() for st in self.stores])
            outs = (_lib.StoreC * n)(*[st.spare().cstruct() for st in self.stores])
            sps = (_lib.SpeciesC * n)(*self._species)
            with _nvtx("advance[all species]"):
                if self.split_advance:
                    wss = (_lib.StoreC * n)(*[st.workspace().cstruct() for st in self.stores])
                    _lib.call("kwb_particles_advance_split", g, n, sps, ins, outs, wss,
                              ctypes.byref(ex.cstruct), E, B, J,
                              jpl.data_ptr() if jpl is not None else None,
                              self.shape_order, self._status.data_ptr(), stream)
                else:
                    _lib.call("kwb_particles_advance_species", g, n, sps, ins, outs,
                              ctypes.byref(ex.cstruct), E, B, J,
                              jpl.data_ptr() if jpl is not None else None,
                              self.shape_order, self._status.data_ptr(), stream)
            with _nvtx("shift[all species]"):
                _lib.call("kwb_particles_shift_species", g, n, outs, ctypes.byref(ex.cstruct),
                          self._status.data_ptr(), stream)
            for st in self.stores:
                st.swap()
            return
        for i, st in enumerate(self.stores):
            src, dst = st.current, st.spare()
            with _nvtx(f"advance[{i}]"):
                if jpl is None:
                    _lib.call("kwb_particles_advance", g, ctypes.byref(self._species[i]),
                              ctypes.byref(src.cstruct()), ctypes.byref(dst.cstruct()),
                              ctypes.byref(ex.cstruct), E, B, J, self.shape_order,
                              self._status[i].data_ptr(), stream)
                else:
                    _lib.call("kwb_particles_advance_zslab", g, ctypes.byref(self._species[i]),
                              ctypes.byref(src.cstruct()), ctypes.byref(dst.cstruct()),
                              ctypes.byref(ex.cstruct), E, B, J, jpl.data_ptr(),
                              self.shape_order, self._status[i].data_ptr(), stream)
            with _nvtx(f"shift[{i}]"):
                _lib.call("kwb_particles_shift", g, ctypes.byref(dst.cstruct()),
                          ctypes.byref(ex.cstruct), self._status[i].data_ptr(), stream)
            st.swap()

    def _undo_particles(self, st):
        """Restore the pre-advance columns and grow what overflowed."""
        for i, store in enumerate(self.stores):
            store.swap()
            if int(st[i, _lib.ST_STORE_OVERFLOW]):
                store.reserve(store.frames_per_sc + int(st[i, _lib.ST_STORE_OVERFLOW]) + 4)
        if int(st[:, _lib.ST_EXCH_OVERFLOW].sum()):
            cap = self._exchange.capacity * 2
            self._exchange = _Exchange(cap, self.stores[0].tdtype, self.device)

    def _enqueue_fields(self):
        with _nvtx("fields"):
            self.update_fields()
        if self.validate:
            g, stream = ctypes.byref(self._grid), self._stream()
            rho_new = self._charge_density_storage()
            _lib.call("kwb_continuity_residual", g, rho_new.data_ptr(), self._rho_prev.data_ptr(),
                      self._J(), self._E(), self._G_prev.data_ptr(), self._resid.data_ptr(), stream)
            self._rho_prev = rho_new

    def _read_status(self):
        self._status_host.copy_(self._status, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return self._status_host.clone()

    def update_fields(self):
        """Yee leapfrog B(1/2) -> E -> B(1/2) with the current J
        (pic/sim.py:164-167)."""
        self.faraday_half()
        self.ampere()
        self.faraday_half()

    def faraday_half(self):
        """B -= dt/2 curl E (pic/kernels.py:253-269, FaradayHalfKernel)."""
        _lib.call("kwb_fields_faraday_half", ctypes.byref(self._grid), self._E(), self._B(),
                  self.params.dt / 2.0, self._stream())

    def ampere(self):
        """E += dt (curl B - J) (pic/kernels.py:272-288, AmpereKernel)."""
        _lib.call("kwb_fields_ampere", ctypes.byref(self._grid), self._E(), self._B(),
                  self._J(), self.params.dt, self._stream())

    def advance_particles(self, zero_j=True):
        """J = 0, then every species' fused advance + shift (the particle
        half of the cycle, pic/sim.py:138-163).  Asynchronous."""
        self._enqueue_particles(zero_j)

    def load_state(self, fields=None, particles=None):
        """Replace fields (name -> (nx, ny, nz) array) and/or particles (one
        dict of canonical records per species: global cx cy cz, ox oy oz,
        ux uy uz, w).  Used for restart and teacher-forced parity runs."""
        if fields:
            for n, a in fields.items():
                self.fields.load_numpy(n, a)
        if particles is not None:
            if len(particles) != len(self.stores):
                raise ValueError("one particle dict per species expected")
            # every species' records on their way before the first load
            # kernel, one synchronisation for all the load checks
            dev = [st.upload(arrays) for st, arrays in zip(self.stores, particles)]
            status = [st.load_packed(d, deferred=True) for st, d in zip(self.stores, dev)]
            bad = torch.stack([s_[_lib.ST_LOAD_ERRORS] for s_ in status if s_ is not None]) \
                if any(s_ is not None for s_ in status) else None
            if bad is not None and int(bad.max()) > 0:
                for st, d, s_ in zip(self.stores, dev, status):
                    if s_ is not None and int(s_[_lib.ST_LOAD_ERRORS]) > 0:
                        st.load_packed(d)   # columns sized from the fullest cell
        self._rho_prev = None
        self._G_prev = None

    def check_status(self):
        """Read the device status words (one small D2H) and raise on any
        contract or capacity violation since the last step; grow stores whose
        fullest column passed GROW_AT of its frames."""
        self._drain_status()
        st = self._read_status()
        self._apply_status(st)
        return st

    def _apply_status(self, st):
        moved = int(st[:, _lib.ST_MOVE_ERRORS].sum())
        if moved:
            raise ContractViolation(
                f"{moved} particle(s) moved a full cell or more before deposit")
        lost = int(st[:, _lib.ST_EXCH_OVERFLOW].sum() + st[:, _lib.ST_STORE_OVERFLOW].sum()
                   + st[:, _lib.ST_LOAD_ERRORS].sum())
        if lost:
            raise AllocationError(
                f"{lost} particle(s) did not fit their cell column or the exchange buffer "
                "(enqueue_step has no redo; use step())")
        guard = int(st[:, _lib.ST_GUARD_OVERFLOW].sum())
        if guard:
            raise AllocationError(
                f"{guard} guard-layer particle(s) exceeded the z-slab exchange message "
                "capacity (DecomposedSimulation.enqueue_step has no redo; use step())")
        for i, store in enumerate(self.stores):
            store.reserve(int(st[i, _lib.ST_MAX_COUNT]))

    def run(self, steps: int):
        for _ in range(steps):
            self.step()

    @property
    def last_residual(self) -> float:
        return float(self._resid[0].item()) if self.step_count else 0.0

    @property
    def last_gauss_drift(self) -> float:
        """max |G^{n+1} - G^n|, G = div E - rho (validate=True only)."""
        return float(self._resid[1].item()) if self.step_count else 0.0

    # -- validation / diagnostics ---------------------------------------------
    def _charge_density_storage(self) -> torch.Tensor:
        nx, ny, nz = self.params.cells.as_tuple()
        rho = torch.zeros((nz, ny, nx), dtype=torch.float64, device=self.device)
        g = ctypes.byref(self._grid)
        for i, st in enumerate(self.stores):
            _lib.call("kwb_charge_density", g, ctypes.byref(self._species[i]),
                      ctypes.byref(st.current.cstruct()), self.shape_order, rho.data_ptr(),
                      self._stream())
        return rho

    def charge_density(self) -> torch.Tensor:
        """float64 charge density, logical (nx, ny, nz) view (pic/sim.py:183-189)."""
        return self._charge_density_storage().permute(2, 1, 0)

    def _moments(self) -> np.ndarray:
        out = torch.zeros((len(self.stores), 3), dtype=torch.float64, device=self.device)
        g = ctypes.byref(self._grid)
        for i, st in enumerate(self.stores):
            _lib.call("kwb_particle_moments", g, ctypes.byref(self._species[i]),
                      ctypes.byref(st.current.cstruct()), out[i].data_ptr(), self._stream())
        return out.cpu().numpy()

    def census(self) -> int:
        return sum(st.census() for st in self.stores)

    def kinetic_energy(self) -> float:
        return float(self._moments()[:, 2].sum())

    def total_charge(self) -> float:
        return float(self._moments()[:, 1].sum())

    def diagnostics(self) -> dict:
        m = self._moments()
        s, max_div_b = field_stats(self.fields)
        f = self.fields
        return {
            "total_charge": float(m[:, 1].sum()),
            "field_energy": 0.5 * s * f.dx * f.dy * f.dz,
            "kinetic_energy": float(m[:, 2].sum()),
            "max_div_b": max_div_b,
            "max_continuity_residual": self.last_residual,
        }

    def total_energy(self) -> float:
        return field_energy(self.fields) + self.kinetic_energy()


def field_stats(fields: YeeFieldSet):
    """(sum of E^2 + B^2, max |div B|) via kwb_field_stats."""
    g = _lib.Grid()
    g.nx, g.ny, g.nz = fields.cells.as_tuple()
    g.scx = g.scy = g.scz = 1
    g.gx, g.gy, g.gz = g.nx, g.ny, g.nz
    g.dtype = _lib.KWB_F32 if fields.dtype == np.float32 else _lib.KWB_F64
    g.dx, g.dy, g.dz, g.dt = fields.dx, fields.dy, fields.dz, 1.0
    out = torch.zeros(2, dtype=torch.float64, device=fields.device)
    E = _lib.ptr3([fields.storage(n) for n in ("Ex", "Ey", "Ez")])
    B = _lib.ptr3([fields.storage(n) for n in ("Bx", "By", "Bz")])
    _lib.call("kwb_field_stats", ctypes.byref(g), E, B, out.data_ptr(),
              torch.cuda.current_stream(fields.device).cuda_stream)
    o = out.cpu().numpy()
    return float(o[0]), float(o[1])


def diagnostics(sim: Simulation) -> dict:
    return sim.diagnostics()


def step(sim: Simulation) -> None:
    sim.step()


def khi_species_particles(params: SimParams, seed: int, sp_i: int, sc_begin: int = 0,
                          sc_end: int | None = None, rng=None):
    """init_khi's particle generation for super cells [sc_begin, sc_end) of
    one species, vectorised (pic/sim.py:239-302).  Returns float64 offsets and
    momenta and int64 global cells, in generation (canonical) order.  Pass the
    same ``rng`` across consecutive chunks to continue the species stream."""
    p = params
    ppc = p.particles_per_cell
    px, py, pz = _near_cubic_factors(ppc)
    sub = np.stack([
        np.tile((np.arange(px) + 0.5) / px, py * pz),
        np.tile(np.repeat((np.arange(py) + 0.5) / py, px), pz),
        np.repeat((np.arange(pz) + 0.5) / pz, px * py),
    ], axis=1)
    scx, scy, scz = p.super_cell.as_tuple()
    grid = p.super_cell_grid
    gx, gy = grid.x, grid.y
    cap = p.frame_capacity
    sc_end = grid.volume if sc_end is None else sc_end
    scs = np.arange(sc_begin, sc_end)
    nsc = scs.shape[0]
    s = np.arange(cap)
    loc = np.stack([s % scx, (s // scx) % scy, s // (scx * scy)], axis=1).astype(np.int64)
    org = np.stack([(scs % gx) * scx, ((scs // gx) % gy) * scy, (scs // (gx * gy)) * scz], axis=1)
    cxyz = org[:, None, :] + loc[None, :, :]
    cx = np.repeat(cxyz[:, :, 0], ppc, axis=1).reshape(-1)
    cy = np.repeat(cxyz[:, :, 1], ppc, axis=1).reshape(-1)
    cz = np.repeat(cxyz[:, :, 2], ppc, axis=1).reshape(-1)
    n_per_sc = cap * ppc
    ox = np.tile(sub[:, 0], cap * nsc)
    oy = np.tile(sub[:, 1], cap * nsc)
    oz = np.tile(sub[:, 2], cap * nsc)
    x_abs = (cx + ox) * p.dx
    v0, amp = p.stream_velocity, p.perturbation
    vx = np.where(cy < p.cells.y // 2, v0, -v0)
    vy = amp * np.sin(2.0 * math.pi * x_abs / (p.cells.x * p.dx))
    vz = np.zeros_like(vx)
    gam = 1.0 / np.sqrt(1.0 - (vx * vx + vy * vy + vz * vz))
    ux, uy, uz = vx * gam, vy * gam, vz * gam
    if p.thermal_u > 0:
        if rng is None:
            rng = np.random.default_rng((seed, sp_i))
        z = rng.normal(0.0, p.thermal_u, 3 * n_per_sc * nsc).reshape(nsc, 3, n_per_sc)
        ux = ux + z[:, 0, :].reshape(-1)
        uy = uy + z[:, 1, :].reshape(-1)
        uz = uz + z[:, 2, :].reshape(-1)
    return dict(cx=cx, cy=cy, cz=cz, ox=ox, oy=oy, oz=oz, ux=ux, uy=uy, uz=uz)


def init_khi(params: SimParams, seed: int = 0, backend=None, strategy="elements",
             validate=True, chunk_super_cells: int = 4096, rng: str = "numpy") -> Simulation:
    """Kelvin-Helmholtz setup (pic/sim.py:239-302): counter-streaming layers
    split along y, sinusoidal v_y perturbation, quiet-start placement,
    thermal jitter; E = B = 0.

    rng="numpy" (default): generated on the host in the reference's exact
    default_rng((seed, species_index)) draw order -- bitwise the reference's
    initial state -- then uploaded.  rng="device": generated in HBM by
    kwb_init_khi (same placement/profile, Philox jitter), for 10^8-10^9
    particles where the host path takes minutes."""
    sim = Simulation(params, backend=backend, strategy=strategy, validate=validate)
    p = params
    if rng == "device":
        for sp_i, store in enumerate(sim.stores):
            store.init_device(p, sp_i, seed)
        return sim
    if rng != "numpy":
        raise ValueError(f"rng must be 'numpy' or 'device', got {rng!r}")
    n_sc = p.super_cell_grid.volume
    dt = p.dtype
    for sp_i, (species, store) in enumerate(zip(p.species, sim.stores)):
        rng = np.random.default_rng((seed, sp_i)) if p.thermal_u > 0 else None
        parts = []
        for b in range(0, n_sc, chunk_super_cells):
            a = khi_species_particles(p, seed, sp_i, b, min(n_sc, b + chunk_super_cells), rng)
            parts.append({k: (v.astype(np.int32) if k in ("cx", "cy", "cz") else v.astype(dt))
                          for k, v in a.items()})
        arrays = {k: np.concatenate([q[k] for q in parts]) for k in parts[0]}
        arrays["w"] = np.full(arrays["cx"].shape, species.weight, dtype=dt)
        store.load_packed(arrays, presorted=True)
    return sim
