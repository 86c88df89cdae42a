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
        a = torch.as_tensor(np.asarray(arr, dtype=self.dtype))
        self._storage[name].copy_(a.permute(2, 1, 0).to(self.device))

    def zero_current(self) -> None:
        self._buf[6:9].zero_()


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


def yee_dispersion_omega(k: float, delta: float, dt: float) -> float:
    """Angular frequency of the discrete vacuum mode along one axis
    (pic/fields.py:172-180)."""
    s = math.sin(k * delta / 2.0) * dt / delta
    if abs(s) > 1.0:
        raise ValueError("mode is evanescent at this dt (CFL violated)")
    return 2.0 * math.asin(s) / dt
