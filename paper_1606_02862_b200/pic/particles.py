"""Super-cell/frame particle store in HBM (API of kernelweave.pic.particles,
reference pic/particles.py:35-211).

Layout -- "cell-column frames" (B200-first, not the reference's linked
lists).  A super cell of V cells (V = frame capacity = 256 by default) owns
K frames of V slots.  Frame k holds the k-th particle of EVERY cell of the
super cell: slot (s, k, c) = (s*K + k)*V + c.  Column (s, c) -- the
particles of local cell c -- fills frames [0, front) from the bottom and
[K-back, K) from the top.  Consequences:

* the particle's cell is implied by its column: no per-particle cell index
  and no occupancy mask are stored (28 B/particle in fp32);
* a warp reading frame k of 32 adjacent cells issues one fully coalesced
  128-B transaction per SoA column;
* the CUDA thread that owns cell c sees only particles of cell c, so the
  Esirkepov current of non-crossing particles accumulates in registers;
* no holes, free stacks or pool overshoot: the reference's ``grow(count)``
  reserves a free frame per leaver (5-32x over-allocation);
  here K only has to exceed the fullest cell.

Two copies of the columns alternate every step: the advance kernel reads one
and writes the other (stayers to the front of their column, in-super-cell
movers to the back of their new column), the shift kernel appends arrivals
from other super cells to the back.  K grows (repack) when a column passes
85% of it.  Canonical order (export/packed) is super cell, then local cell,
then frame; the reference orders by frame chain and slot within a super
cell, so comparisons are order-independent within a super cell (SURVEY.md
§8b).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from .. import _lib
from ..errors import AllocationError, ContractViolation
from ..workdiv import Extent3, linearize_3d
from .fields import TORCH_DTYPE
from .pusher import MacroParticle

FLOAT_COLUMNS = ("ox", "oy", "oz", "ux", "uy", "uz", "w")
PACKED_FIELDS = ("cx", "cy", "cz", "ox", "oy", "oz", "ux", "uy", "uz", "w")
HEADROOM = 1.5
GROW_AT = 0.85


def initial_frames(max_col: int, mean_col: float) -> int:
    """Frames per super cell for a fresh store: room for the fullest cell
    and for the spread a thermal plasma develops (cell counts drift towards
    Poisson statistics, and the fullest of ~10^6-10^7 cells in a thermal
    plasma has been measured 6.5 sigma above the mean -- 57-60 particles at
    25 ppc, tools/occupancy_trace.py), with margin so that growth -- a
    repack plus large allocations -- stays out of steady-state stepping.
    The store is a few GB against 180 GB of HBM: spend memory, not time."""
    return max(8, math.ceil(max_col * 1.3) + 4,
               math.ceil(mean_col + 10.0 * math.sqrt(max(mean_col, 1.0))) + 8)


class _Columns:
    __slots__ = ("ox", "oy", "oz", "ux", "uy", "uz", "w", "front", "back", "frames")

    def __init__(self, n_sc, cells, frames, tdtype, device):
        n = n_sc * frames * cells
        for c in FLOAT_COLUMNS:   # slots outside [0, front) and [K-back, K) are never read
            setattr(self, c, torch.empty(n, dtype=tdtype, device=device))
        self.front = torch.zeros(n_sc * cells, dtype=torch.int32, device=device)
        self.back = torch.zeros(n_sc * cells, dtype=torch.int32, device=device)
        self.frames = frames

    def cstruct(self) -> _lib.StoreC:
        s = _lib.StoreC()
        for c in FLOAT_COLUMNS + ("front", "back"):
            setattr(s, c, getattr(self, c).data_ptr())
        s.frames_per_sc = self.frames
        return s


class SuperCellStore:
    """Per-species particle store: cell-column frames per super cell."""

    def __init__(self, cells, super_cell, dtype=np.float64, device="cuda", frames_per_sc: int = 4):
        self.cells = Extent3.of(cells)
        self.super_cell = Extent3.of(super_cell)
        self.sc_grid = Extent3(self.cells.x // self.super_cell.x,
                               self.cells.y // self.super_cell.y,
                               self.cells.z // self.super_cell.z)
        self.n_super_cells = self.sc_grid.volume
        self.capacity = self.super_cell.volume
        if self.capacity > 256:
            raise ContractViolation(
                f"super-cell volume {self.capacity} > 256: one CUDA thread owns one cell")
        self.dtype = np.dtype(dtype)
        self.tdtype = TORCH_DTYPE[self.dtype]
        self.device = torch.device(device)
        self.frames_per_sc = max(1, int(frames_per_sc))
        self._cols = [self._new_columns(), None]
        self.loaded = 0  # particles at the last load (sizes exchange buffers without a sync)

    # -- storage --------------------------------------------------------------
    def _new_columns(self) -> _Columns:
        return _Columns(self.n_super_cells, self.capacity, self.frames_per_sc, self.tdtype,
                        self.device)

    def _reset_columns(self) -> None:
        """Empty columns of frames_per_sc frames for a fresh load: buffers of
        that size are reused (a restart keeps its ~GB allocations), others
        are reallocated."""
        keep = [c for c in self._cols if c is not None and c.frames == self.frames_per_sc]
        if keep:
            keep[0].front.zero_()
            keep[0].back.zero_()
            self._cols = [keep[0], keep[1] if len(keep) > 1 else None]
        else:
            self._cols = [self._new_columns(), None]

    @property
    def current(self) -> _Columns:
        return self._cols[0]

    def spare(self) -> _Columns:
        """The write target of the next advance (allocated on first use)."""
        if self._cols[1] is None or self._cols[1].frames != self.frames_per_sc:
            self._cols[1] = self._new_columns()
        return self._cols[1]

    def swap(self) -> None:
        self._cols.reverse()

    def workspace(self) -> _Columns:
        """Scratch columns of the split advance (kwb_particles_advance_split:
        new offsets, momenta and carries per slot), sized like the store."""
        ws = getattr(self, "_ws", None)
        if ws is None or ws.frames != self.frames_per_sc:
            self._ws = ws = self._new_columns()
        return ws

    def reserve(self, max_column: int, stream=None) -> bool:
        """Grow frames_per_sc so the fullest column sits below GROW_AT of it;
        repacks the live particles on the device.  Returns True if it grew."""
        if max_column <= GROW_AT * self.frames_per_sc:
            return False
        old = self.current
        self.frames_per_sc = max(math.ceil(max_column * HEADROOM) + 8, self.frames_per_sc + 1)
        new = self._new_columns()
        g = self._grid_struct()
        _lib.call("kwb_store_repack", _lib.ctypes.byref(g), _lib.ctypes.byref(old.cstruct()),
                  _lib.ctypes.byref(new.cstruct()), _stream(stream, self.device))
        self._cols = [new, None]
        return True

    def _grid_struct(self) -> _lib.Grid:
        g = _lib.Grid()
        g.nx, g.ny, g.nz = self.cells.as_tuple()
        g.scx, g.scy, g.scz = self.super_cell.as_tuple()
        g.gx, g.gy, g.gz = self.sc_grid.as_tuple()
        g.dtype = _lib.KWB_F32 if self.dtype == np.float32 else _lib.KWB_F64
        g.dx = g.dy = g.dz = 1.0
        g.dt = 1.0
        return g

    # -- reference-shaped views ---------------------------------------------------
    @property
    def n_frames(self) -> int:
        return self.n_super_cells * self.frames_per_sc

    def _col2d(self, name):
        return getattr(self.current, name).view(self.n_frames, self.capacity)

    ox = property(lambda self: self._col2d("ox"))
    oy = property(lambda self: self._col2d("oy"))
    oz = property(lambda self: self._col2d("oz"))
    ux = property(lambda self: self._col2d("ux"))
    uy = property(lambda self: self._col2d("uy"))
    uz = property(lambda self: self._col2d("uz"))
    w = property(lambda self: self._col2d("w"))

    @property
    def column_counts(self) -> torch.Tensor:
        """Particles per cell column, (n_super_cells, capacity) int32."""
        c = self.current
        return (c.front + c.back).view(self.n_super_cells, self.capacity)

    @property
    def count(self) -> torch.Tensor:
        """Particles per super cell (device int32)."""
        return self.column_counts.sum(dim=1, dtype=torch.int32)

    @property
    def occ(self) -> torch.Tensor:
        """Slot occupancy (n_frames, capacity) uint8, as the reference's occ."""
        c = self.current
        K, V = self.frames_per_sc, self.capacity
        k = torch.arange(K, device=self.device).view(1, K, 1)
        f = c.front.view(-1, 1, V)
        b = c.back.view(-1, 1, V)
        m = (k < f) | (k >= K - b)
        return m.to(torch.uint8).view(self.n_frames, V)

    @property
    def nfilled(self) -> torch.Tensor:
        """Particles per frame (n_frames,), as the reference's nfilled."""
        return self.occ.sum(dim=1, dtype=torch.int32)

    @property
    def owner(self) -> torch.Tensor:
        """Owning super cell per frame, -1 for empty frames."""
        sc = torch.arange(self.n_super_cells, device=self.device, dtype=torch.int32)
        own = sc.repeat_interleave(self.frames_per_sc)
        return torch.where(self.nfilled > 0, own, torch.full_like(own, -1))

    def super_cell_of(self, cell) -> int:
        sc = (cell[0] // self.super_cell.x, cell[1] // self.super_cell.y,
              cell[2] // self.super_cell.z)
        return linearize_3d(sc, self.sc_grid)

    def frames_of(self, sc: int):
        """Frame indices of one super cell that hold particles, in order."""
        nf = self.nfilled[sc * self.frames_per_sc:(sc + 1) * self.frames_per_sc].cpu().numpy()
        return [sc * self.frames_per_sc + k for k in range(self.frames_per_sc) if nf[k] > 0]

    def census(self) -> int:
        c = self.current
        return int((c.front.sum(dtype=torch.int64) + c.back.sum(dtype=torch.int64)).item())

    def super_cell_counts(self) -> np.ndarray:
        return self.count.cpu().numpy().astype(np.int64)

    # -- host <-> device ------------------------------------------------------------
    def packed(self, fields=PACKED_FIELDS, stream=None, out=None) -> dict:
        """Canonical-order records (super cell, cell, frame) as host numpy
        arrays: global cells int32, storage-type floats (export kernel).
        `out` (optional): dict of preallocated host tensors (pinned for an
        asynchronous DMA) with at least census() elements each; the result
        arrays are views of them."""
        dev = self.packed_device(stream)
        if out is None:
            return {n: dev[n].cpu().numpy() for n in fields}
        n = dev["cx"].shape[0]
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        res = {}
        with torch.cuda.stream(s):
            for f in fields:
                dst = out[f]
                if dst.numel() < n:
                    raise ValueError(f"packed: out[{f!r}] holds {dst.numel()} < {n} records")
                dst[:n].copy_(dev[f], non_blocking=True)
                res[f] = dst[:n]
        s.synchronize()
        return {f: v.numpy() for f, v in res.items()}

    def packed_device(self, stream=None, columns=None, clear=False) -> dict:
        """Export (device tensors) the particles of all columns, or of the
        column range `columns` = (begin, end); clear=True empties them."""
        c0, c1 = columns if columns is not None else (0, self.current.front.numel())
        cnt = (self.current.front[c0:c1] + self.current.back[c0:c1]).to(torch.int64)
        start = torch.zeros(cnt.numel() + 1, dtype=torch.int64, device=self.device)
        torch.cumsum(cnt, 0, out=start[1:])
        n = int(start[-1].item())
        m = max(n, 1)  # never hand the C ABI a NULL buffer (clear with no particles)
        out = {c: torch.empty(m, dtype=torch.int32, device=self.device) for c in ("cx", "cy", "cz")}
        for c in FLOAT_COLUMNS:
            out[c] = torch.empty(m, dtype=self.tdtype, device=self.device)
        if n or clear:
            g = self._grid_struct()
            _lib.call("kwb_store_export", _lib.ctypes.byref(g),
                      _lib.ctypes.byref(self.current.cstruct()), c0, c1, start.data_ptr(),
                      int(bool(clear)), out["cx"].data_ptr(), out["cy"].data_ptr(),
                      out["cz"].data_ptr(), _lib.ptr7([out[c] for c in FLOAT_COLUMNS]),
                      _stream(stream, self.device))
        return {k: v[:n] for k, v in out.items()}

    def column_starts(self, columns):
        """Exclusive prefix sum (device, int64, length n+1) of the particle
        counts of the column range `columns` = (begin, end)."""
        c0, c1 = columns
        cnt = (self.current.front[c0:c1] + self.current.back[c0:c1]).to(torch.int64)
        start = torch.zeros(cnt.numel() + 1, dtype=torch.int64, device=self.device)
        torch.cumsum(cnt, 0, out=start[1:])
        return start

    def export_into(self, columns, start, ints, flts, offset=0, clear=False, stream=None):
        """kwb_store_export of the column range into rows of caller buffers:
        ints (3, m) int32 (cx, cy, cz) and flts (7, m) storage-type
        (ox oy oz ux uy uz w), records placed from column `offset`; `start`
        from column_starts().  No host synchronisation."""
        c0, c1 = columns
        g = self._grid_struct()
        isz, fsz = ints.element_size(), flts.element_size()
        ip = [ints.data_ptr() + (k * ints.stride(0) + offset) * isz for k in range(3)]
        fp = [flts.data_ptr() + (k * flts.stride(0) + offset) * fsz for k in range(7)]
        _lib.call("kwb_store_export", _lib.ctypes.byref(g),
                  _lib.ctypes.byref(self.current.cstruct()), c0, c1, start.data_ptr(),
                  int(bool(clear)), ip[0], ip[1], ip[2],
                  _lib.Ptr7(*fp), _stream(stream, self.device))

    def extract_into(self, columns, start, ints, flts, count_out, status, capacity,
                     offset=0, stream=None):
        """kwb_store_extract: move the particles of the column range into rows
        of caller buffers (from column `offset`, at most `capacity` records,
        all or nothing); the count lands in count_out (device int64)."""
        c0, c1 = columns
        g = self._grid_struct()
        isz, fsz = ints.element_size(), flts.element_size()
        ip = [ints.data_ptr() + (k * ints.stride(0) + offset) * isz for k in range(3)]
        fp = [flts.data_ptr() + (k * flts.stride(0) + offset) * fsz for k in range(7)]
        _lib.call("kwb_store_extract", _lib.ctypes.byref(g),
                  _lib.ctypes.byref(self.current.cstruct()), c0, c1, start.data_ptr(), capacity,
                  ip[0], ip[1], ip[2], _lib.Ptr7(*fp), count_out.data_ptr(), status.data_ptr(),
                  _stream(stream, self.device))

    def append_counted(self, ints, flts, count, capacity, status, offset=0, stream=None):
        """kwb_store_load_counted: append min(count, capacity) records held in
        rows of (3, m) int32 / (7, m) buffers from column `offset`; `count` is
        a device int64 (no host synchronisation)."""
        g = self._grid_struct()
        isz, fsz = ints.element_size(), flts.element_size()
        ip = [ints.data_ptr() + (k * ints.stride(0) + offset) * isz for k in range(3)]
        fp = [flts.data_ptr() + (k * flts.stride(0) + offset) * fsz for k in range(7)]
        _lib.call("kwb_store_load_counted", _lib.ctypes.byref(g),
                  _lib.ctypes.byref(self.current.cstruct()), count.data_ptr(), capacity,
                  ip[0], ip[1], ip[2], _lib.Ptr7(*fp), status.data_ptr(),
                  _stream(stream, self.device))

    def append(self, arrays: dict, stream=None, status=None) -> None:
        """Append particle records (device tensors or host arrays; global
        cells in this store's grid) to their columns without resizing.
        Records that do not fit are counted in status[ST_LOAD_ERRORS] (the
        caller's status words, checked with the step's status)."""
        def up(a, tdt):
            t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))
            return t.to(device=self.device, dtype=tdt, non_blocking=True).contiguous()
        d_cells = [up(arrays[c], torch.int32) for c in ("cx", "cy", "cz")]
        n = d_cells[0].shape[0]
        if n == 0:
            return
        d_f = [up(arrays[c], self.tdtype) for c in FLOAT_COLUMNS]
        if status is None:
            status = torch.zeros(_lib.STATUS_WORDS, dtype=torch.int32, device=self.device)
        g = self._grid_struct()
        _lib.call("kwb_store_load", _lib.ctypes.byref(g), _lib.ctypes.byref(self.current.cstruct()),
                  n, d_cells[0].data_ptr(), d_cells[1].data_ptr(), d_cells[2].data_ptr(),
                  _lib.ptr7(d_f), status.data_ptr(), _stream(stream, self.device))

    def upload(self, arrays: dict) -> dict:
        """The records of `arrays` as device tensors of the store's types
        (asynchronous from pinned host memory)."""
        def up(a, tdt):
            t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))
            return t.to(device=self.device, dtype=tdt, non_blocking=True).contiguous()
        d = {c: up(arrays[c], torch.int32) for c in ("cx", "cy", "cz")}
        d.update({c: up(arrays[c], self.tdtype) for c in FLOAT_COLUMNS})
        return d

    def load_packed(self, arrays: dict, stream=None, presorted: bool = False,
                    deferred: bool = False):
        """Replace the store's content with particle records (global cells
        cx/cy/cz plus ox oy oz ux uy uz w; host numpy or device tensors).
        Columns are sized from the fullest cell with headroom; the load
        kernel appends every record to its column.  deferred=True: return
        the device status words instead of checking them (the caller checks
        several stores with one synchronisation and reloads a failed one
        with deferred=False)."""
        del presorted  # any order is accepted
        d = self.upload(arrays)
        d_cells = [d[c] for c in ("cx", "cy", "cz")]
        d_f = [d[c] for c in FLOAT_COLUMNS]
        n = d_cells[0].shape[0]
        nx, ny, nz = self.cells.as_tuple()
        if n:
            ext = torch.stack([t for c in d_cells for t in torch.aminmax(c)]).cpu()
            lo, hi = ext[0::2], ext[1::2]
            if int(lo.min()) < 0 or int(hi[0]) >= nx or int(hi[1]) >= ny or int(hi[2]) >= nz:
                raise ContractViolation("particle cell index outside the grid")
        # size the columns from the mean load (Poisson headroom, initial_frames);
        # only if some column overflows is the fullest cell counted and the
        # load redone (a histogram over all cells costs more than the load)
        max_col = 0
        for _attempt in range(2):
            self.frames_per_sc = initial_frames(max_col, n / (nx * ny * nz))
            self.loaded = n
            self._reset_columns()
            status = torch.zeros(_lib.STATUS_WORDS, dtype=torch.int32, device=self.device)
            g = self._grid_struct()
            _lib.call("kwb_store_load", _lib.ctypes.byref(g),
                      _lib.ctypes.byref(self.current.cstruct()), n, d_cells[0].data_ptr(),
                      d_cells[1].data_ptr(), d_cells[2].data_ptr(), _lib.ptr7(d_f),
                      status.data_ptr(), _stream(stream, self.device))
            if deferred:
                return status
            bad = int(status[_lib.ST_LOAD_ERRORS].item())
            if not bad:
                return
            cx, cy, cz = (c.to(torch.int64) for c in d_cells)
            cell = (cz * ny + cy) * nx + cx
            max_col = int(torch.bincount(cell, minlength=nx * ny * nz).max().item())
        raise AllocationError(f"{bad} particle record(s) could not be loaded")

    def init_device(self, params, species_index: int, seed: int, offsets=(0, 0, 0),
                    global_cells=None, stream=None) -> None:
        """Fill the store with init_khi's quiet-start particles on the device
        (kwb_init_khi): same placement and velocity profile as the host path,
        thermal jitter from Philox instead of numpy's default_rng."""
        from .sim import _near_cubic_factors
        ppc = params.particles_per_cell
        px, py, pz = _near_cubic_factors(ppc)
        n_cells = self.cells.volume
        self.frames_per_sc = initial_frames(ppc, float(ppc))
        self._reset_columns()
        gx, gy = (global_cells or self.cells.as_tuple())[:2]
        ini = _lib.InitC(ppc=ppc, px=px, py=py, pz=pz,
                         stream_velocity=params.stream_velocity,
                         perturbation=params.perturbation, thermal_u=params.thermal_u,
                         weight=params.species[species_index].weight,
                         seed=int(seed) & 0xFFFFFFFFFFFFFFFF, species_index=species_index,
                         x_offset=offsets[0], y_offset=offsets[1], z_offset=offsets[2],
                         global_nx=gx, global_ny=gy)
        g = self._grid_struct()
        g.dx, g.dy, g.dz = params.dx, params.dy, params.dz
        _lib.call("kwb_init_khi", _lib.ctypes.byref(g), _lib.ctypes.byref(ini),
                  _lib.ctypes.byref(self.current.cstruct()), _stream(stream, self.device))
        self.loaded = n_cells * ppc

    def insert(self, p: MacroParticle) -> None:
        """Append one particle to its cell column (host-side path,
        pic/particles.py:129-144)."""
        cnt = int(self.column_counts.max().item())
        self.reserve(cnt + 1)
        rec = {"cx": [p.cell[0]], "cy": [p.cell[1]], "cz": [p.cell[2]],
               "ox": [p.offset[0]], "oy": [p.offset[1]], "oz": [p.offset[2]],
               "ux": [p.u[0]], "uy": [p.u[1]], "uz": [p.u[2]], "w": [p.weight]}
        d_cells = [torch.tensor(rec[c], dtype=torch.int32, device=self.device)
                   for c in ("cx", "cy", "cz")]
        d_f = [torch.tensor(rec[c], dtype=self.tdtype, device=self.device) for c in FLOAT_COLUMNS]
        status = torch.zeros(_lib.STATUS_WORDS, dtype=torch.int32, device=self.device)
        g = self._grid_struct()
        _lib.call("kwb_store_load", _lib.ctypes.byref(g), _lib.ctypes.byref(self.current.cstruct()),
                  1, d_cells[0].data_ptr(), d_cells[1].data_ptr(), d_cells[2].data_ptr(),
                  _lib.ptr7(d_f), status.data_ptr(), _stream(None, self.device))
        if int(status[_lib.ST_LOAD_ERRORS].item()):
            raise AllocationError("insert: particle could not be stored")
        self.loaded += 1

    def iter_particles(self):
        """(sc, frame, slot, MacroParticle) in canonical order."""
        pk = self.packed()
        c = self.current
        front = c.front.cpu().numpy()
        back = c.back.cpu().numpy()
        K, V = self.frames_per_sc, self.capacity
        i = 0
        for col in range(front.shape[0]):
            s, cell = divmod(col, V)
            f, b = int(front[col]), int(back[col])
            for j in range(f + b):
                k = j if j < f else K - b + (j - f)
                yield s, s * K + k, cell, MacroParticle(
                    (int(pk["cx"][i]), int(pk["cy"][i]), int(pk["cz"][i])),
                    (float(pk["ox"][i]), float(pk["oy"][i]), float(pk["oz"][i])),
                    (float(pk["ux"][i]), float(pk["uy"][i]), float(pk["uz"][i])),
                    float(pk["w"][i]))
                i += 1

    def check_integrity(self):
        """Columns fit their frames and do not overlap; occupancy sums to the
        census (the reference's chain/ownership/occupancy checks,
        pic/particles.py:188-211, restated for the column layout; membership
        is structural: a particle's cell is its column)."""
        c = self.current
        assert int(c.front.min().item()) >= 0 and int(c.back.min().item()) >= 0
        assert int((c.front + c.back).max().item()) <= self.frames_per_sc, "column overflow"
        assert int(self.occ.sum().item()) == self.census(), "occupancy != census"
        return True


def _stream(stream, device):
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream
