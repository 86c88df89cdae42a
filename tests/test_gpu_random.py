"""Randomised one-step parity of the CUDA path against the oracle: random
grid and super-cell shapes, cell sizes, dtypes, shapes (CIC/TSC/PCS), 1-3
species with random charge/mass/weight, random particles (offsets include
the exact 0.0 / 1.0 edge values, momenta up to ~0.9 cell per step) and
random E/B fields.  From identical state, one step: particle records
bitwise, fields within the stated one-step bar (1e-13 f64 / 1e-6 f32),
charge conservation on both sides."""

import numpy as np
import pytest

from golden_util import rel_l2
from parity_util import FIELDS9, TOL_1STEP, assert_particles_bitwise, check_fields, order_spread

pytestmark = pytest.mark.gpu

SUPER_CELLS = [(8, 8, 4), (4, 4, 4), (4, 8, 2), (8, 4, 4)]


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    sc = SUPER_CELLS[seed % len(SUPER_CELLS)]
    cells = tuple(int(s * rng.integers(1, 4)) for s in sc)
    dtype = np.float32 if seed % 2 == 0 else np.float64
    shape = ("cic", "tsc", "pcs")[seed % 3]
    deltas = tuple(float(d) for d in rng.uniform(0.7, 1.3, 3))
    n_sp = int(rng.integers(1, 4))
    species = []
    for i in range(n_sp):
        species.append((f"s{i}", float(rng.choice([-1.0, 1.0]) * rng.uniform(0.5, 2.0)),
                        float(rng.uniform(0.5, 50.0)), float(rng.uniform(0.05, 0.5))))
    return rng, sc, cells, dtype, shape, deltas, species


def _particles(rng, cells, n, dtype, dt, deltas):
    c = np.stack([rng.integers(0, cells[a], n) for a in range(3)], 1).astype(np.int32)
    o = rng.random((n, 3))
    edge = rng.random((n, 3)) < 0.03
    o[edge] = rng.choice([0.0, 1.0], size=int(edge.sum()))
    o = o.astype(dtype)
    if dtype == np.float32:
        o = np.minimum(o, np.float32(1.0))
    # |v| dt / delta <= 0.9 on every axis: u with |u| < 0.9 min(delta)/dt / sqrt(3) ... capped
    vmax = min(0.95, 0.9 * min(deltas) / dt)
    v = rng.uniform(-1.0, 1.0, (n, 3))
    v *= vmax / np.sqrt(3.0) * rng.random((n, 1))
    gam = 1.0 / np.sqrt(1.0 - (v * v).sum(1, keepdims=True))
    u = (v * gam).astype(dtype)
    return dict(cx=c[:, 0], cy=c[:, 1], cz=c[:, 2], ox=o[:, 0], oy=o[:, 1], oz=o[:, 2],
                ux=u[:, 0], uy=u[:, 1], uz=u[:, 2])


@pytest.mark.parametrize("seed", range(32))
def test_random_one_step_vs_oracle(seed):
    from oracle.pic import OracleSim
    from paper_1606_02862_b200.pic import SimParams, Simulation, Species
    rng, sc, cells, dtype, shape, deltas, species = _case(seed)
    p = SimParams(cells=cells, species=tuple(Species(*s) for s in species), dtype=dtype,
                  shape=shape, super_cell=sc, dx=deltas[0], dy=deltas[1], dz=deltas[2])
    gpu = Simulation(p, validate=True)
    orc = OracleSim(p, validate=True, shape_order=p.shape_order, threads=2)
    # random fields (J zero): the gather and push see non-trivial E and B
    fields = {}
    for n in FIELDS9:
        a = np.zeros(cells, dtype=dtype) if n.startswith("J") else \
            (0.05 * rng.standard_normal(cells)).astype(dtype)
        fields[n] = a
        getattr(orc.fields, n)[...] = a
    recs = []
    for (_, _, _, w) in species:
        n = int(rng.integers(50, 400))
        r = _particles(rng, cells, n, dtype, float(p.dt), deltas)
        r["w"] = np.full(n, w, dtype=dtype)
        recs.append(r)
    gpu.load_state(fields=fields, particles=recs)
    for st, rec in zip(orc.stores, recs):
        scx, scy, scz = st.super_cell
        gx, gy, _ = st.sc_grid
        cx, cy, cz = (np.asarray(rec[k]).astype(np.int64) for k in ("cx", "cy", "cz"))
        scid = cx // scx + gx * (cy // scy + gy * (cz // scz))
        o = np.argsort(scid, kind="stable")
        st.load_packed(scid[o], {k: np.asarray(v)[o] for k, v in rec.items()})
    spread = order_spread(orc)
    gpu.step()
    orc.step()
    for gs, os_ in zip(gpu.stores, orc.stores):
        assert_particles_bitwise(gs, os_)
    check_fields(f"random{seed}", gpu.fields, lambda n: getattr(orc.fields, n),
                 TOL_1STEP[np.dtype(dtype)], spread=spread)
    lim = 1e-12 if dtype == np.float64 else 1e-6
    assert gpu.last_residual <= lim
