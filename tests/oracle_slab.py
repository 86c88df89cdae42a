"""Oracle-backed stand-in for one slab's local Simulation (TEST
INFRASTRUCTURE).  It exposes the interface DecomposedSimulation drives
(fields.storage, stores[i].packed_device/append, advance_particles,
faraday_half, ampere, ...) on top of oracle.pic, so the z-slab exchange logic
can be exercised on CPU with the gloo backend and compared with a
single-domain oracle run."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from oracle import pic as orc

COLS = ("ox", "oy", "oz", "ux", "uy", "uz", "w")


class _Fields:
    def __init__(self, of):
        self.of = of

    def storage(self, name):
        return torch.from_numpy(getattr(self.of, name)).permute(2, 1, 0)

    def numpy(self, name):
        return getattr(self.of, name).copy()


class _Store:
    def __init__(self, st: orc.OracleStore, dtype):
        self.st = st
        gx, gy, gz = st.sc_grid
        self.sc_grid = type("G", (), {"x": gx, "y": gy, "z": gz})()
        self.capacity = st.capacity
        self.tdtype = torch.float32 if dtype == np.float32 else torch.float64

    def census(self):
        return self.st.census()

    def packed(self):
        return self.st.packed()

    def packed_device(self, columns, clear):
        V = self.capacity
        s0, s1 = columns[0] // V, columns[1] // V
        st = self.st
        rec = {k: [] for k in ("cx", "cy", "cz") + COLS}
        for sc in range(s0, s1):
            for f in st.frames_of(sc):
                for s in np.nonzero(st.occ[f])[0]:
                    for k in rec:
                        rec[k].append(getattr(st, k)[f, s])
                if clear:
                    st.occ[f, :] = 0
                    st.nfilled[f] = 0
        if clear:
            lib = orc.lib()
            lib.orc_unlink_empty(ctypes.byref(st._cpool()), st.n_super_cells)
        out = {}
        for k, v in rec.items():
            dt = np.int32 if k in ("cx", "cy", "cz") else st.dtype
            out[k] = torch.from_numpy(np.asarray(v, dtype=dt))
        return out

    def column_starts(self, columns):
        """Only the total ([-1]) is used by the decomposition."""
        V = self.capacity
        st = self.st
        n = sum(int(st.occ[f].sum()) for sc in range(columns[0] // V, columns[1] // V)
                for f in st.frames_of(sc))
        return torch.tensor([0, n], dtype=torch.int64)

    def export_into(self, columns, start, ints, flts, offset=0, clear=False):
        rec = self.packed_device(columns, clear)
        n = rec["cx"].shape[0]
        for k, c in enumerate(("cx", "cy", "cz")):
            ints[k, offset:offset + n] = rec[c]
        for k, c in enumerate(COLS):
            flts[k, offset:offset + n] = rec[c]

    def append(self, rec, status=None):
        st = self.st
        n = rec["cx"].shape[0]
        for i in range(n):
            cell = (int(rec["cx"][i]), int(rec["cy"][i]), int(rec["cz"][i]))
            scx, scy, scz = st.super_cell
            gx, gy, _ = st.sc_grid
            sc = cell[0] // scx + gx * (cell[1] // scy + gy * (cell[2] // scz))
            f = int(st.tail[sc])
            if f >= 0 and st.nfilled[f] < st.capacity:
                slot = int(np.argmin(st.occ[f]))
            else:
                f = st.alloc_frame(sc)
                slot = 0
            st.occ[f, slot] = 1
            st.nfilled[f] += 1
            st.cx[f, slot], st.cy[f, slot], st.cz[f, slot] = cell
            for k in COLS:
                getattr(st, k)[f, slot] = rec[k][i].item()


class OracleLocal:
    """One slab on the CPU oracle."""

    def __init__(self, params):
        self.sim = orc.OracleSim(params, validate=False, shape_order=params.shape_order, threads=2)
        self.params = params
        self.fields = _Fields(self.sim.fields)
        self.stores = [_Store(s, self.sim.dtype) for s in self.sim.stores]
        self.device = torch.device("cpu")
        self._status = torch.zeros((len(self.stores), 8), dtype=torch.int32)
        self.step_count = 0

    # lagged status hooks of the GPU Simulation: nothing to do on CPU
    def _drain_status(self, keep=0):
        pass

    def _post_status(self):
        pass

    def check_status(self):
        assert int(self._status.sum()) == 0

    def census(self):
        return self.sim.census()

    def load_state(self, fields=None, particles=None):
        if fields:
            for n, a in fields.items():
                setattr(self.sim.fields, n, np.ascontiguousarray(np.asarray(a, dtype=self.sim.dtype)))
        if particles is not None:
            for st, rec in zip(self.sim.stores, particles):
                scx, scy, scz = st.super_cell
                gx, gy, _ = st.sc_grid
                cx, cy, cz = (np.asarray(rec[k]).astype(np.int64) for k in ("cx", "cy", "cz"))
                sc = cx // scx + gx * (cy // scy + gy * (cz // scz))
                order = np.argsort(sc, kind="stable")
                st.load_packed(sc[order], {k: np.asarray(v)[order] for k, v in rec.items()})

    def advance_particles(self):
        s = self.sim
        f = s.fields
        f.Jx[:] = 0
        f.Jy[:] = 0
        f.Jz[:] = 0
        cf = f._cfields()
        nx, ny, nz = s.cells
        for i, st in enumerate(s.stores):
            cs = st._cstore()
            s._fn("gather")(ctypes.byref(cs), ctypes.byref(cf), s.threads)
            s._fn("push")(ctypes.byref(cs), s.qm[i], s.threads)
            s._fn("move")(ctypes.byref(cs), *s.move_k, nx, ny, nz, s.threads)
            tiles = s._tiles_for(st.n_super_cells)
            err = s._fn("deposit")(ctypes.byref(cs), ctypes.byref(cf), s.shape_order,
                                   orc._p(s.fac[i]), *s.super_cell, orc._p(tiles), s.threads)
            assert err == 0
        for st in s.stores:
            orc.migrate(st)

    def faraday_half(self):
        s = self.sim
        s._fn("faraday")(ctypes.byref(s.fields._cfields()), s.params.dt / 2.0, s.threads)

    def ampere(self):
        s = self.sim
        s._fn("ampere")(ctypes.byref(s.fields._cfields()), s.params.dt, s.threads)
