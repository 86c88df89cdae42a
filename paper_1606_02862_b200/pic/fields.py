"""Yee lattice fields on the device (API of kernelweave.pic.fields,
reference pic/fields.py:1-180).

Staggering (cell units, particle position = cell index + offset):

    rho[i,j,k] at (i+1/2, j+1/2, k+1/2)
    Ex,Jx at (i+1, j+1/2, k+1/2)   Bx at (i+1/2, j+1, k+1)
    Ey,Jy at (i+1/2, j+1, k+1/2)   By at (i+1, j+1/2, k+1)
    Ez,Jz at (i+1/2, j+1/2, k+1)   Bz at (i+1, j+1, k+1/2)

HBM layout: each lattice is ONE contiguous torch tensor stored x fastest,
``storage[k, j, i]`` -- z-planes are contiguous, which is what the z-slab
domain decomposition exchanges.  ``fields.Ex`` etc. are the logical
(nx, ny, nz) views (``storage.permute(2, 1, 0)``), indexed exactly like the
reference's numpy arrays.  All nine lattices live in one allocation.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from ..workdiv import Extent3

STAGGER = {
    "Ex": (1.0, 0.5, 0.5),
    "Ey": (0.5, 1.0, 0.5),
    "Ez": (0.5, 0.5, 1.0),
    "Bx": (0.5, 1.0, 1.0),
    "By": (1.0, 0.5, 1.0),
    "Bz": (1.0, 1.0, 0.5),
}

E_COMPONENTS = ("Ex", "Ey", "Ez")
B_COMPONENTS = ("Bx", "By", "Bz")
J_COMPONENTS = ("Jx", "Jy", "Jz")
ALL_COMPONENTS = E_COMPONENTS + B_COMPONENTS + J_COMPONENTS

TORCH_DTYPE = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}


class YeeFieldSet:
    """E, B, J lattices over a periodic cell grid, resident in HBM."""

    def __init__(self, cells, dx=1.0, dy=1.0, dz=1.0, dtype=np.float64, device="cuda"):
        self.cells = Extent3.of(cells)
        self.dx, self.dy, self.dz = float(dx), float(dy), float(dz)
        self.dtype = np.dtype(dtype)
        self.device = torch.device(device)
        nx, ny, nz = self.cells.as_tuple()
        self._buf = torch.zeros((9, nz, ny, nx), dtype=TORCH_DTYPE[self.dtype],
                                device=self.device)
        self._storage = {n: self._buf[i] for i, n in enumerate(ALL_COMPONENTS)}

    @property
    def shape(self):
        return self.cells.as_tuple()

    def storage(self, name: str) -> torch.Tensor:
        """Contiguous (nz, ny, nx) tensor of one lattice (x fastest)."""
        return self._storage[name]

    def components(self, names=ALL_COMPONENTS):
        return tuple(getattr(self, n) for n in names)

    def copy(self) -> "YeeFieldSet":
        out = YeeFieldSet(self.cells, self.dx, self.dy, self.dz, self.dtype, self.device)
        out._buf.copy_(self._buf)
        return out

    def numpy(self, name: str) -> np.ndarray:
        """Host copy of one lattice in the reference's (nx, ny, nz) C order."""
        return np.ascontiguousarray(getattr(self, name).cpu().numpy())

    def load_numpy(self, name: str, arr) -> None:
        """Upload a reference-ordered (nx, ny, nz) host array into one lattice."""
        if isinstance(arr, torch.Tensor):
            a = arr.to(TORCH_DTYPE[self.dtype])   # no copy if the dtype matches
        else:
            a = torch.as_tensor(np.ascontiguousarray(arr, dtype=self.dtype))
        # copy as laid out (pinned host memory: asynchronous DMA), transpose
        # to x-fastest on the device
        d = a.to(self.device, non_blocking=True)
        self._storage[name].copy_(d.permute(2, 1, 0))

    def zero_current(self) -> None:
        """J = 0 on the current stream (kwb_zero_step)."""
        import ctypes

        from .. import _lib
        _lib.call("kwb_zero_step", ctypes.byref(_grid_of(self)),
                  ctypes.cast(_ptr3(self, J_COMPONENTS), ctypes.c_void_p), None, 0,
                  torch.cuda.current_stream(self.device).cuda_stream)


def _component_property(name):
    def get(self):
        return self._storage[name].permute(2, 1, 0)

    def set(self, value):
        v = torch.as_tensor(value, device=self.device)
        self._storage[name].copy_(v.permute(2, 1, 0) if v.dim() == 3 else v)

    return property(get, set, doc=f"{name} as a logical (nx, ny, nz) view")


for _n in ALL_COMPONENTS:
    setattr(YeeFieldSet, _n, _component_property(_n))


def tsc_weights(offset: float):
    """Quadratic-spline (TSC) weights over left/center/right cells
    (pic/fields.py:66-77); host helper, compensated centre weight."""
    if not 0.0 <= offset < 1.0:
        raise ValueError(f"offset {offset} outside [0, 1)")
    o = offset - 0.5
    wl = 0.5 * (0.5 - o) ** 2
    wr = 0.5 * (0.5 + o) ** 2
    return wl, 1.0 - wl - wr, wr


def _dm(a, dim):
    return a - torch.roll(a, 1, dims=dim)


def _dp(a, dim):
    return torch.roll(a, -1, dims=dim) - a


def div_b(fields: YeeFieldSet) -> torch.Tensor:
    """Discrete face divergence of B (pic/fields.py:145-151), (nx, ny, nz) view."""
    return (_dp(fields.Bx, 0) / fields.dx + _dp(fields.By, 1) / fields.dy
            + _dp(fields.Bz, 2) / fields.dz)


def div_j(fields: YeeFieldSet) -> torch.Tensor:
    """Discrete divergence of J at the charge sites (pic/fields.py:154-160)."""
    return (_dm(fields.Jx, 0) / fields.dx + _dm(fields.Jy, 1) / fields.dy
            + _dm(fields.Jz, 2) / fields.dz)


def field_energy(fields: YeeFieldSet) -> float:
    """Sum over cells of (|E|^2 + |B|^2)/2 times the cell volume
    (pic/fields.py:163-169), reduced on the device by kwb_field_stats."""
    from .sim import field_stats
    s, _ = field_stats(fields)
    return 0.5 * s * fields.dx * fields.dy * fields.dz


def _grid_of(fields: YeeFieldSet):
    from .. import _lib
    g = _lib.Grid()
    g.nx, g.ny, g.nz = fields.cells.as_tuple()
    g.scx = g.scy = g.scz = 1
    g.gx, g.gy, g.gz = g.nx, g.ny, g.nz
    g.dtype = _lib.KWB_F32 if fields.dtype == np.float32 else _lib.KWB_F64
    g.dx, g.dy, g.dz, g.dt = fields.dx, fields.dy, fields.dz, 0.0
    return g


def _ptr3(fields, names):
    from .. import _lib
    return _lib.ptr3([fields.storage(n) for n in names])


def yee_update_b(fields: YeeFieldSet, half_dt: float) -> None:
    """B <- B - half_dt * curl E (pic/fields.py:127-133) on the device, by
    the same kernel as Simulation's Faraday half step (kwb_fields_faraday_half,
    the compiled reference recipe pic/kernels.py:253-269 -- bit for bit the
    reference's float64 result; in float32 the reference's whole-grid numpy
    helper rounds differently and the kernel recipe is the one step() uses).
    Asynchronous on the current stream."""
    import ctypes

    from .. import _lib
    _lib.call("kwb_fields_faraday_half", ctypes.byref(_grid_of(fields)),
              _ptr3(fields, E_COMPONENTS), _ptr3(fields, B_COMPONENTS), float(half_dt),
              torch.cuda.current_stream(fields.device).cuda_stream)


def yee_update_e(fields: YeeFieldSet, dt: float) -> None:
    """E <- E + dt * (curl B - J) (pic/fields.py:136-142) on the device
    (kwb_fields_ampere, pic/kernels.py:272-288).  Asynchronous."""
    import ctypes

    from .. import _lib
    _lib.call("kwb_fields_ampere", ctypes.byref(_grid_of(fields)),
              _ptr3(fields, E_COMPONENTS), _ptr3(fields, B_COMPONENTS),
              _ptr3(fields, J_COMPONENTS), float(dt),
              torch.cuda.current_stream(fields.device).cuda_stream)


def gather_fields(fields: YeeFieldSet, p):
    """(E, B) at a particle (pic/fields.py:95-118): trilinear interpolation of
    the Yee-staggered lattices, evaluated on the device by kwb_fields_gather
    with the advance kernel's recipe (double arithmetic, periodic wrap,
    rounded to the storage type -- the values the reference's compiled
    gather hands its push, pic/kernels.py:53-77).  ``p`` is a MacroParticle
    (returns two length-3 arrays) or a sequence of them (returns (n, 3)
    arrays).  Synchronises to return host arrays."""
    import ctypes

    from .. import _lib
    single = hasattr(p, "cell")
    ps = [p] if single else list(p)
    n = len(ps)
    cells = torch.tensor([list(q.cell) for q in ps] or [[0, 0, 0]], dtype=torch.int32,
                         device=fields.device)
    offs = torch.tensor([list(q.offset) for q in ps] or [[0.0, 0.0, 0.0]], dtype=torch.float64,
                        device=fields.device)
    out = torch.empty((max(n, 1), 6), dtype=fields.storage("Ex").dtype, device=fields.device)
    _lib.call("kwb_fields_gather", ctypes.byref(_grid_of(fields)),
              _ptr3(fields, E_COMPONENTS), _ptr3(fields, B_COMPONENTS), ctypes.c_int64(n),
              _lib.ptr(cells), _lib.ptr(offs), _lib.ptr(out),
              torch.cuda.current_stream(fields.device).cuda_stream)
    h = out[:n].cpu().numpy()
    if single:
        return h[0, :3].copy(), h[0, 3:].copy()
    return h[:, :3].copy(), h[:, 3:].copy()


def yee_dispersion_omega(k: float, delta: float, dt: float) -> float:
    """Angular frequency of the discrete vacuum mode along one axis
    (pic/fields.py:172-180)."""
    s = math.sin(k * delta / 2.0) * dt / delta
    if abs(s) > 1.0:
        raise ValueError("mode is evanescent at this dt (CFL violated)")
    return 2.0 * math.asin(s) / dt
