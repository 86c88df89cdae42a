"""CPU oracle of the kernelweave.pic cycle -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  It is the checker the CUDA
path is compared against and the CPU timing port; the product package never
imports it.

It restates the reference (``/root/reference/pkg/src/kernelweave/pic``):

* ``OracleStore`` mirrors ``SuperCellStore`` (pic/particles.py:35-211): the
  same frame pool, doubly linked chains, free stack and doubling ``grow``, so
  canonical particle order, frame ids and the pool-order ``_rho_tsc`` sum
  are reproduced exactly.
* ``OracleSim.step`` mirrors ``Simulation.step`` (pic/sim.py:134-176); the
  per-particle and per-cell arithmetic runs in ``liborcpic.so``
  (oracle/pic_oracle.c), which follows the Numba kernels' rounding recipe.
* ``oracle_init_khi`` is a vectorised restatement of ``init_khi``
  (pic/sim.py:239-328) with the same ``default_rng((seed, sp_i))`` draw order.

Deposit shapes: order 2 (TSC) is the reference; orders 1 (CIC) and 3 (PCS)
are the SURVEY.md §8c extension (same decomposition, other shape function,
7-point arrays and a 3-cell tile halo for PCS).

Pinned bitwise against golden dumps of the unmodified reference:
tests/golden/make_golden.py -> tests/golden/*.npz, tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liborcpic.so")

FLOAT_FIELDS = ("ox", "oy", "oz", "ux", "uy", "uz", "w",
                "epx", "epy", "epz", "bpx", "bpy", "bpz", "oox", "ooy", "ooz")
INT_FIELDS = ("cx", "cy", "cz", "ocx", "ocy", "ocz")
PACKED_FIELDS = ("cx", "cy", "cz", "ox", "oy", "oz", "ux", "uy", "uz", "w")


class _Store(ctypes.Structure):
    _fields_ = [("n_sc", ctypes.c_int64), ("cap", ctypes.c_int64),
                ("head", ctypes.c_void_p), ("next_f", ctypes.c_void_p),
                ("occ", ctypes.c_void_p)] + \
        [(n, ctypes.c_void_p) for n in FLOAT_FIELDS[:7]] + \
        [(n, ctypes.c_void_p) for n in FLOAT_FIELDS[7:]] + \
        [(n, ctypes.c_void_p) for n in INT_FIELDS]


class _Fields(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dz", ctypes.c_double)] + \
        [(n, ctypes.c_void_p) for n in
         ("Ex", "Ey", "Ez", "Bx", "By", "Bz", "Jx", "Jy", "Jz")]


class _Pool(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("head", "tail", "next_f", "prev_f", "owner", "nfilled",
                 "free_stack", "free_top")]


_lib = None


def build(force: bool = False) -> str:
    """Compile liborcpic.so with oracle/Makefile (gcc, no FMA contraction)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.orc_div_rcp_check.argtypes = [I64, ctypes.c_uint64]
        L.orc_div_rcp_check.restype = I64
        L.orc_div6_check.argtypes = [I64, ctypes.c_uint64]
        L.orc_div6_check.restype = I64
        L.orc_set_merge_seed.argtypes = [ctypes.c_uint64]
        L.orc_set_reverse_slots.argtypes = [ctypes.c_int]
        for sfx in ("_f32", "_f64"):
            getattr(L, "orc_gather" + sfx).argtypes = [P, P, I]
            getattr(L, "orc_push" + sfx).argtypes = [P, D, I]
            getattr(L, "orc_move" + sfx).argtypes = [P, D, D, D, I64, I64, I64, I]
            f = getattr(L, "orc_deposit" + sfx)
            f.argtypes = [P, P, I, P, I64, I64, I64, P, I]
            f.restype = I64
            getattr(L, "orc_faraday" + sfx).argtypes = [P, D, I]
            getattr(L, "orc_ampere" + sfx).argtypes = [P, D, I]
            getattr(L, "orc_rho" + sfx).argtypes = [P, I64, P, I, D, P, I64, I64, I64]
            getattr(L, "orc_apply_migration" + sfx).argtypes = [P, P, I64, P, P, P]
        L.orc_scan_leavers.argtypes = [P, P, I64, I64, I64, I64, I64, P, P, P]
        L.orc_scan_leavers.restype = I64
        L.orc_unlink_empty.argtypes = [P, I64]
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    assert a.flags.c_contiguous
    return a.ctypes.data


def default_threads() -> int:
    return int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1))


def near_cubic_factors(n: int) -> tuple[int, int, int]:
    """pic/sim.py:36-52 (deterministic balanced factorisation)."""
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


class OracleStore:
    """Restatement of SuperCellStore (pic/particles.py:35-118, 146-211)."""

    def __init__(self, cells, super_cell, dtype=np.float64, initial_frames=16):
        self.cells = tuple(int(c) for c in cells)
        self.super_cell = tuple(int(s) for s in super_cell)
        self.sc_grid = tuple(c // s for c, s in zip(self.cells, self.super_cell))
        self.n_super_cells = self.sc_grid[0] * self.sc_grid[1] * self.sc_grid[2]
        self.capacity = self.super_cell[0] * self.super_cell[1] * self.super_cell[2]
        self.dtype = np.dtype(dtype)
        f = max(4, initial_frames)
        for n in FLOAT_FIELDS:
            setattr(self, n, np.zeros((f, self.capacity), dtype=self.dtype))
        for n in INT_FIELDS:
            setattr(self, n, np.zeros((f, self.capacity), dtype=np.int32))
        self.occ = np.zeros((f, self.capacity), dtype=np.uint8)
        self.next_f = np.full(f, -1, dtype=np.int32)
        self.prev_f = np.full(f, -1, dtype=np.int32)
        self.owner = np.full(f, -1, dtype=np.int32)
        self.nfilled = np.zeros(f, dtype=np.int32)
        self.head = np.full(self.n_super_cells, -1, dtype=np.int32)
        self.tail = np.full(self.n_super_cells, -1, dtype=np.int32)
        self.free_stack = np.arange(f - 1, -1, -1, dtype=np.int32)
        self.free_top = np.array([f], dtype=np.int64)

    @property
    def n_frames(self) -> int:
        return self.next_f.shape[0]

    @property
    def free_frames(self) -> int:
        return int(self.free_top[0])

    def grow(self, min_free: int):
        """pic/particles.py:72-101: double the pool until min_free frames are free."""
        while self.free_frames < min_free:
            old = self.n_frames
            new = old * 2
            for n in FLOAT_FIELDS + INT_FIELDS + ("occ",):
                a = getattr(self, n)
                b = np.zeros((new, self.capacity), dtype=a.dtype)
                b[:old] = a
                setattr(self, n, b)
            for n, fill in (("next_f", -1), ("prev_f", -1), ("owner", -1), ("nfilled", 0)):
                a = getattr(self, n)
                b = np.full(new, fill, dtype=np.int32)
                b[:old] = a
                setattr(self, n, b)
            stack = np.zeros(new, dtype=np.int32)
            top = self.free_frames
            stack[:top] = self.free_stack[:top]
            stack[top: top + (new - old)] = np.arange(new - 1, old - 1, -1, dtype=np.int32)
            self.free_stack = stack
            self.free_top[0] = top + (new - old)

    def alloc_frame(self, sc: int) -> int:
        """pic/particles.py:103-118."""
        if self.free_frames == 0:
            self.grow(1)
        self.free_top[0] -= 1
        f = int(self.free_stack[self.free_top[0]])
        self.owner[f] = sc
        self.next_f[f] = -1
        self.nfilled[f] = 0
        tail = int(self.tail[sc])
        self.prev_f[f] = tail
        if tail >= 0:
            self.next_f[tail] = f
        else:
            self.head[sc] = f
        self.tail[sc] = f
        return f

    def frames_of(self, sc: int):
        out, f = [], int(self.head[sc])
        while f >= 0:
            out.append(f)
            f = int(self.next_f[f])
        return out

    def census(self) -> int:
        return int(self.occ.sum())

    def canonical_index(self):
        """(frame, slot) arrays in canonical order (pic/particles.py:8-10)."""
        fi, si = [], []
        for sc in range(self.n_super_cells):
            for f in self.frames_of(sc):
                s = np.nonzero(self.occ[f])[0]
                fi.append(np.full(s.shape, f, dtype=np.int64))
                si.append(s.astype(np.int64))
        if not fi:
            return np.zeros(0, np.int64), np.zeros(0, np.int64)
        return np.concatenate(fi), np.concatenate(si)

    def packed(self, fields=PACKED_FIELDS):
        fi, si = self.canonical_index()
        return {n: getattr(self, n)[fi, si] for n in fields}

    def super_cell_counts(self) -> np.ndarray:
        cnt = np.zeros(self.n_super_cells, dtype=np.int64)
        live = self.owner >= 0
        np.add.at(cnt, self.owner[live], self.nfilled[live])
        return cnt

    # -- ctypes views -------------------------------------------------------
    def _cstore(self) -> _Store:
        s = _Store()
        s.n_sc, s.cap = self.n_super_cells, self.capacity
        s.head, s.next_f, s.occ = _p(self.head), _p(self.next_f), _p(self.occ)
        for n in FLOAT_FIELDS + INT_FIELDS:
            setattr(s, n, _p(getattr(self, n)))
        return s

    def _cpool(self) -> _Pool:
        p = _Pool()
        for n in ("head", "tail", "next_f", "prev_f", "owner", "nfilled",
                  "free_stack", "free_top"):
            setattr(p, n, _p(getattr(self, n)))
        return p

    def load_packed(self, sc_of: np.ndarray, arrays: dict):
        """Fill an empty store densely from canonical-order arrays (sc_of
        ascending), as _bulk_fill does at init (pic/sim.py:305-328)."""
        n_sc = self.n_super_cells
        counts = np.bincount(sc_of, minlength=n_sc)
        cap = self.capacity
        start = 0
        for sc in range(n_sc):
            n = int(counts[sc])
            frames = (n + cap - 1) // cap
            self.grow(frames)
            for k in range(frames):
                f = self.alloc_frame(sc)
                a, b = start + k * cap, start + min((k + 1) * cap, n)
                cnt = b - a
                for name in PACKED_FIELDS:
                    getattr(self, name)[f, :cnt] = arrays[name][a:b]
                self.occ[f, :cnt] = 1
                self.nfilled[f] = cnt
            start += n


def migrate(store: OracleStore) -> int:
    """pic/particles.py:316-345 `migrate_particles`."""
    L = lib()
    bound = max(1, store.census())
    out_f = np.empty(bound, np.int32)
    out_s = np.empty(bound, np.int32)
    out_d = np.empty(bound, np.int32)
    scx, scy, scz = store.super_cell
    gx, gy, _ = store.sc_grid
    cs = store._cstore()
    count = L.orc_scan_leavers(ctypes.byref(cs), _p(store.nfilled), scx, scy, scz, gx, gy,
                               _p(out_f), _p(out_s), _p(out_d))
    if count:
        store.grow(count)
        cs = store._cstore()
        pl = store._cpool()
        sfx = "_f32" if store.dtype == np.float32 else "_f64"
        getattr(L, "orc_apply_migration" + sfx)(ctypes.byref(cs), ctypes.byref(pl), count,
                                                _p(out_f), _p(out_s), _p(out_d))
    pl = store._cpool()
    L.orc_unlink_empty(ctypes.byref(pl), store.n_super_cells)
    return int(count)


class OracleFields:
    """YeeFieldSet restatement (pic/fields.py:39-63): (nx, ny, nz), z fastest."""

    NAMES = ("Ex", "Ey", "Ez", "Bx", "By", "Bz", "Jx", "Jy", "Jz")

    def __init__(self, cells, dx, dy, dz, dtype):
        self.cells = tuple(int(c) for c in cells)
        self.dx, self.dy, self.dz = float(dx), float(dy), float(dz)
        self.dtype = np.dtype(dtype)
        for n in self.NAMES:
            setattr(self, n, np.zeros(self.cells, dtype=self.dtype))

    def _cfields(self) -> _Fields:
        f = _Fields()
        f.nx, f.ny, f.nz = self.cells
        f.dx, f.dy, f.dz = self.dx, self.dy, self.dz
        for n in self.NAMES:
            setattr(f, n, _p(getattr(self, n)))
        return f


def div_j(f: OracleFields) -> np.ndarray:
    """pic/fields.py:154-160 (numpy, storage-type arithmetic)."""
    def dm(a, ax):
        return a - np.roll(a, 1, axis=ax)
    return dm(f.Jx, 0) / f.dx + dm(f.Jy, 1) / f.dy + dm(f.Jz, 2) / f.dz


def div_b(f: OracleFields) -> np.ndarray:
    """pic/fields.py:145-151."""
    def dp(a, ax):
        return np.roll(a, -1, axis=ax) - a
    return dp(f.Bx, 0) / f.dx + dp(f.By, 1) / f.dy + dp(f.Bz, 2) / f.dz


def field_energy(f: OracleFields) -> float:
    """pic/fields.py:163-169."""
    total = 0.0
    for n in ("Ex", "Ey", "Ez", "Bx", "By", "Bz"):
        total += float(np.sum(getattr(f, n).astype(np.float64) ** 2))
    return 0.5 * total * f.dx * f.dy * f.dz


class OracleSim:
    """Restatement of Simulation (pic/sim.py:55-228) over liborcpic."""

    def __init__(self, params, validate=True, shape_order=2, threads=None):
        p = params
        self.params = p
        self.validate = validate
        self.shape_order = int(shape_order)
        self.threads = threads or default_threads()
        self.merge_seed = 0   # 0: Serial tile-merge order; else BlockPool-like permutation
        self.reverse_slots = False   # particle order inside tiles (order-spread only)
        self.step_count = 0
        self.last_residual = 0.0
        cells = tuple(p.cells)
        self.cells = cells
        self.super_cell = tuple(p.super_cell)
        self.dtype = np.dtype(p.dtype)
        self.fields = OracleFields(cells, p.dx, p.dy, p.dz, self.dtype)
        self.stores = [OracleStore(cells, self.super_cell, self.dtype) for _ in p.species]
        deltas = (p.dx, p.dy, p.dz)
        vol = p.dx * p.dy * p.dz
        self.vol = vol
        self.qm = [s.charge * p.dt / (2.0 * s.mass) for s in p.species]
        self.fac = [np.array([-s.charge * deltas[a] / (p.dt * vol) for a in range(3)],
                             dtype=np.float64) for s in p.species]
        self.move_k = (p.dt / p.dx, p.dt / p.dy, p.dt / p.dz)
        self._rho_prev = None
        self._tiles = None
        self._sfx = "_f32" if self.dtype == np.float32 else "_f64"

    def _fn(self, name):
        return getattr(lib(), "orc_" + name + self._sfx)

    def _tiles_for(self, n_sc):
        hw = 3 if self.shape_order == 3 else 2
        sc = self.super_cell
        size = n_sc * 3 * (sc[0] + 2 * hw) * (sc[1] + 2 * hw) * (sc[2] + 2 * hw)
        if self._tiles is None or self._tiles.size != size:
            self._tiles = np.zeros(size, dtype=self.dtype)
        return self._tiles

    def step(self):
        p, f = self.params, self.fields
        if self.validate and self._rho_prev is None:
            self._rho_prev = self.charge_density()
        f.Jx[:] = 0
        f.Jy[:] = 0
        f.Jz[:] = 0
        cf = f._cfields()
        nt = self.threads
        nx, ny, nz = self.cells
        for i, st in enumerate(self.stores):
            cs = st._cstore()
            self._fn("gather")(ctypes.byref(cs), ctypes.byref(cf), nt)
            self._fn("push")(ctypes.byref(cs), self.qm[i], nt)
            self._fn("move")(ctypes.byref(cs), *self.move_k, nx, ny, nz, nt)
            tiles = self._tiles_for(st.n_super_cells)
            lib().orc_set_merge_seed(self.merge_seed + 7919 * i if self.merge_seed else 0)
            lib().orc_set_reverse_slots(1 if self.reverse_slots else 0)
            err = self._fn("deposit")(ctypes.byref(cs), ctypes.byref(cf), self.shape_order,
                                      _p(self.fac[i]), *self.super_cell, _p(tiles), nt)
            if err:
                raise RuntimeError(
                    f"{err} particle(s) moved a full cell or more before deposit")
        for st in self.stores:
            migrate(st)
        self._fn("faraday")(ctypes.byref(cf), p.dt / 2.0, nt)
        self._fn("ampere")(ctypes.byref(cf), p.dt, nt)
        self._fn("faraday")(ctypes.byref(cf), p.dt / 2.0, nt)
        if self.validate:
            rho_new = self.charge_density()
            residual = np.abs((rho_new - self._rho_prev) / p.dt
                              + div_j(f).astype(np.float64)).max()
            self.last_residual = float(residual)
            self._rho_prev = rho_new
        self.step_count += 1

    def run(self, steps):
        for _ in range(steps):
            self.step()

    def charge_density(self) -> np.ndarray:
        rho = np.zeros(self.cells, dtype=np.float64)
        for sp, st in zip(self.params.species, self.stores):
            cs = st._cstore()
            self._fn("rho")(ctypes.byref(cs), st.n_frames, _p(st.owner), self.shape_order,
                            sp.charge / self.vol, _p(rho), *self.cells)
        return rho

    def census(self) -> int:
        return sum(s.census() for s in self.stores)

    def kinetic_energy(self) -> float:
        """pic/sim.py:194-207."""
        total = 0.0
        for sp, st in zip(self.params.species, self.stores):
            m = st.occ != 0
            if not m.any():
                continue
            ux = st.ux[m].astype(np.float64)
            uy = st.uy[m].astype(np.float64)
            uz = st.uz[m].astype(np.float64)
            gam = np.sqrt(1.0 + ux * ux + uy * uy + uz * uz)
            total += sp.mass * float(np.sum((gam - 1.0) * st.w[m].astype(np.float64)))
        return total

    def total_charge(self) -> float:
        total = 0.0
        for sp, st in zip(self.params.species, self.stores):
            m = st.occ != 0
            total += sp.charge * float(st.w[m].astype(np.float64).sum())
        return total

    def diagnostics(self) -> dict:
        return {
            "total_charge": self.total_charge(),
            "field_energy": field_energy(self.fields),
            "kinetic_energy": self.kinetic_energy(),
            "max_div_b": float(np.abs(div_b(self.fields)).max()),
            "max_continuity_residual": self.last_residual,
        }


def khi_particles(params, seed: int, sp_i: int):
    """Vectorised restatement of init_khi's per-species particle generation
    (pic/sim.py:239-302).  Returns canonical-order arrays (super cells
    ascending, generation order) as float64 momenta/offsets before the
    storage cast, plus the per-particle super-cell index."""
    p = params
    ppc = p.particles_per_cell
    px, py, pz = near_cubic_factors(ppc)
    sub = np.stack([
        np.tile((np.arange(px) + 0.5) / px, py * pz),
        np.tile(np.repeat((np.arange(py) + 0.5) / py, px), pz),
        np.repeat((np.arange(pz) + 0.5) / pz, px * py),
    ], axis=1)
    scx, scy, scz = tuple(p.super_cell)
    nx, ny, nz = tuple(p.cells)
    gx, gy, gz = nx // scx, ny // scy, nz // scz
    cap = scx * scy * scz
    n_sc = gx * gy * gz
    half_y = ny // 2
    lx_len = nx * p.dx
    s = np.arange(cap)
    loc = np.stack([s % scx, (s // scx) % scy, s // (scx * scy)], axis=1).astype(np.int64)
    scs = np.arange(n_sc)
    org = np.stack([(scs % gx) * scx, ((scs // gx) % gy) * scy, (scs // (gx * gy)) * scz], axis=1)
    n_per_sc = cap * ppc
    cells_xyz = (org[:, None, :] + loc[None, :, :])           # (n_sc, cap, 3)
    cx = np.repeat(cells_xyz[:, :, 0], ppc, axis=1).reshape(-1)
    cy = np.repeat(cells_xyz[:, :, 1], ppc, axis=1).reshape(-1)
    cz = np.repeat(cells_xyz[:, :, 2], ppc, axis=1).reshape(-1)
    ox = np.tile(sub[:, 0], cap * n_sc)
    oy = np.tile(sub[:, 1], cap * n_sc)
    oz = np.tile(sub[:, 2], cap * n_sc)
    x_abs = (cx + ox) * p.dx
    v0, amp = p.stream_velocity, p.perturbation
    vx = np.where(cy < half_y, v0, -v0)
    vy = amp * np.sin(2.0 * math.pi * x_abs / lx_len)
    vz = np.zeros_like(vx)
    gam = 1.0 / np.sqrt(1.0 - (vx * vx + vy * vy + vz * vz))
    ux, uy, uz = vx * gam, vy * gam, vz * gam
    if p.thermal_u > 0:
        rng = np.random.default_rng((seed, sp_i))
        z = rng.normal(0.0, p.thermal_u, 3 * n_per_sc * n_sc).reshape(n_sc, 3, n_per_sc)
        ux = ux + z[:, 0, :].reshape(-1)
        uy = uy + z[:, 1, :].reshape(-1)
        uz = uz + z[:, 2, :].reshape(-1)
    sc_of = np.repeat(scs, n_per_sc)
    return sc_of, dict(cx=cx, cy=cy, cz=cz, ox=ox, oy=oy, oz=oz, ux=ux, uy=uy, uz=uz)


def oracle_init_khi(params, seed=0, validate=True, shape_order=2, threads=None) -> OracleSim:
    """init_khi restatement (pic/sim.py:239-302) into an OracleSim."""
    sim = OracleSim(params, validate=validate, shape_order=shape_order, threads=threads)
    dt = sim.dtype
    for sp_i, (species, store) in enumerate(zip(params.species, sim.stores)):
        sc_of, a = khi_particles(params, seed, sp_i)
        arrays = {k: (v.astype(np.int32) if k in ("cx", "cy", "cz") else v.astype(dt))
                  for k, v in a.items()}
        arrays["w"] = np.full(sc_of.shape, species.weight, dtype=dt)
        store.load_packed(sc_of, arrays)
    return sim
