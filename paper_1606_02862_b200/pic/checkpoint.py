"""KWPIC1 checkpoint: the flat binary dump SPEC.md:541 specifies (and the
reference never implements) -- "magic KWPIC1, extents, species table, then
field arrays x-fastest, then particle records per super cell".

Layout (little endian):

    b"KWPIC1\\0\\0"                                   8 bytes
    u32 version (=1), u32 float bytes (4|8)
    i32 nx ny nz scx scy scz
    f64 dx dy dz dt
    u32 shape order, u32 n_species, u64 step_count
    f64 stream_velocity perturbation thermal_u, i32 particles_per_cell, i32 pad
    per species: 32-byte utf-8 name, f64 charge mass weight
    9 field arrays Ex Ey Ez Bx By Bz Jx Jy Jz, nx*ny*nz floats each, x fastest
    per species: u64 n, u32 count per super cell (ascending), then n records
        {i32 cx, cy, cz; F ox, oy, oz, ux, uy, uz, w} in canonical order:
        super cell ascending, within it (cell, ox, oy, oz, ux, uy, uz, w)
        ascending by value bits -- so identical states give identical files
        regardless of slot order (SPEC.md:592 determinism).
"""

from __future__ import annotations

import struct

import numpy as np

MAGIC = b"KWPIC1\0\0"
NAMES = ("Ex", "Ey", "Ez", "Bx", "By", "Bz", "Jx", "Jy", "Jz")
REC = ("cx", "cy", "cz", "ox", "oy", "oz", "ux", "uy", "uz", "w")


def _canonical(pk: dict, p) -> tuple[np.ndarray, dict]:
    scx, scy, scz = p.super_cell.as_tuple()
    g = p.super_cell_grid
    cx, cy, cz = (np.asarray(pk[k]).astype(np.int64) for k in ("cx", "cy", "cz"))
    sc = cx // scx + g.x * (cy // scy + g.y * (cz // scz))
    cell = (cz * p.cells.y + cy) * p.cells.x + cx
    keys = []
    for k in reversed(REC[3:]):
        a = np.asarray(pk[k])
        keys.append(a.view(np.uint64 if a.itemsize == 8 else np.uint32))
    keys += [cell, sc]
    order = np.lexsort(keys)
    counts = np.bincount(sc, minlength=g.volume).astype(np.uint32)
    return counts, {k: np.asarray(pk[k])[order] for k in REC}


def _field_numpy(sim, name) -> np.ndarray:
    """(nx, ny, nz) host copy of one lattice (device Simulation or any object
    whose fields are numpy arrays, e.g. the test oracle)."""
    f = sim.fields
    return f.numpy(name) if hasattr(f, "numpy") else np.asarray(getattr(f, name))


def save_checkpoint(sim, path: str) -> None:
    """Write a Simulation's state as KWPIC1."""
    p = sim.params
    F = np.dtype(p.dtype)
    nx, ny, nz = p.cells.as_tuple()
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<II", 1, F.itemsize))
        fh.write(struct.pack("<6i", nx, ny, nz, *p.super_cell.as_tuple()))
        fh.write(struct.pack("<4d", p.dx, p.dy, p.dz, p.dt))
        fh.write(struct.pack("<IIQ", p.shape_order, len(p.species), sim.step_count))
        fh.write(struct.pack("<3dii", p.stream_velocity, p.perturbation, p.thermal_u,
                             p.particles_per_cell, 0))
        for s in p.species:
            fh.write(s.name.encode()[:32].ljust(32, b"\0"))
            fh.write(struct.pack("<3d", s.charge, s.mass, s.weight))
        for n in NAMES:
            a = _field_numpy(sim, n).astype(F.newbyteorder("<"), copy=False)
            fh.write(np.ascontiguousarray(a.transpose(2, 1, 0)).tobytes())   # x fastest
        rec_dt = np.dtype([("cx", "<i4"), ("cy", "<i4"), ("cz", "<i4")] +
                          [(k, F.newbyteorder("<")) for k in REC[3:]])
        for st in sim.stores:
            counts, pk = _canonical(st.packed(), p)
            n = int(counts.sum())
            fh.write(struct.pack("<Q", n))
            fh.write(counts.astype("<u4").tobytes())
            rec = np.empty(n, dtype=rec_dt)
            for k in REC:
                rec[k] = pk[k]
            fh.write(rec.tobytes())


def read_checkpoint(path: str) -> dict:
    """Parse a KWPIC1 file into host arrays (no GPU needed)."""
    with open(path, "rb") as fh:
        buf = fh.read()
    if buf[:8] != MAGIC:
        raise ValueError(f"{path}: not a KWPIC1 checkpoint")
    off = 8
    version, fb = struct.unpack_from("<II", buf, off); off += 8
    if version != 1:
        raise ValueError(f"unsupported KWPIC1 version {version}")
    nx, ny, nz, scx, scy, scz = struct.unpack_from("<6i", buf, off); off += 24
    dx, dy, dz, dt = struct.unpack_from("<4d", buf, off); off += 32
    order, n_sp, step = struct.unpack_from("<IIQ", buf, off); off += 16
    v0, amp, uth, ppc, _ = struct.unpack_from("<3dii", buf, off); off += 32
    species = []
    for _ in range(n_sp):
        name = buf[off:off + 32].rstrip(b"\0").decode(); off += 32
        q, m, w = struct.unpack_from("<3d", buf, off); off += 24
        species.append((name, q, m, w))
    F = np.dtype("<f4" if fb == 4 else "<f8")
    ncell = nx * ny * nz
    fields = {}
    for n in NAMES:
        a = np.frombuffer(buf, dtype=F, count=ncell, offset=off).reshape(nz, ny, nx)
        fields[n] = np.ascontiguousarray(a.transpose(2, 1, 0))   # reference (nx, ny, nz) order
        off += ncell * fb
    n_sc = (nx // scx) * (ny // scy) * (nz // scz)
    rec_dt = np.dtype([("cx", "<i4"), ("cy", "<i4"), ("cz", "<i4")] + [(k, F) for k in REC[3:]])
    particles = []
    for _ in range(n_sp):
        (n,) = struct.unpack_from("<Q", buf, off); off += 8
        counts = np.frombuffer(buf, dtype="<u4", count=n_sc, offset=off).copy(); off += 4 * n_sc
        rec = np.frombuffer(buf, dtype=rec_dt, count=n, offset=off); off += n * rec_dt.itemsize
        particles.append({k: np.ascontiguousarray(rec[k]) for k in REC} | {"_counts": counts})
    return dict(cells=(nx, ny, nz), super_cell=(scx, scy, scz), deltas=(dx, dy, dz), dt=dt,
                shape_order=order, species=species, step_count=step, stream_velocity=v0,
                perturbation=amp, thermal_u=uth, particles_per_cell=ppc,
                dtype=np.dtype(np.float32 if fb == 4 else np.float64), fields=fields,
                particles=particles)


def load_checkpoint(path: str, backend=None, validate=True):
    """Rebuild a Simulation from a KWPIC1 file (restart)."""
    from .params import SHAPES, SimParams, Species
    from .sim import Simulation
    c = read_checkpoint(path)
    shape = {v: k for k, v in SHAPES.items()}[c["shape_order"]]
    p = SimParams(cells=c["cells"], dx=c["deltas"][0], dy=c["deltas"][1], dz=c["deltas"][2],
                  dt=c["dt"], species=tuple(Species(*s) for s in c["species"]),
                  particles_per_cell=c["particles_per_cell"], super_cell=c["super_cell"],
                  dtype=c["dtype"], stream_velocity=c["stream_velocity"],
                  perturbation=c["perturbation"], thermal_u=c["thermal_u"], shape=shape)
    sim = Simulation(p, backend=backend, validate=validate)
    sim.load_state(fields=c["fields"],
                   particles=[{k: v for k, v in d.items() if k != "_counts"}
                              for d in c["particles"]])
    sim.step_count = c["step_count"]
    return sim
