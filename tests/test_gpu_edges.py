"""Edge cases of the CUDA path against the oracle (bitwise particle state after
one step from identical state, fields within tolerance):

* empty store, a single particle, one particle per cell;
* offsets exactly 0 and exactly 1.0 (the f32 rounding case the reference
  keeps), particles on super-cell faces;
* near-light-speed momenta (the largest per-step displacement CFL allows);
* a grid that is a single super cell along an axis (periodic self-wrap, the
  super-cell shift returns the particle to the same super cell);
* non-default super cells ((4,4,4): 64 threads per CTA), anisotropic cells;
* PCS and CIC in float64.
"""

import numpy as np
import pytest

from golden_util import rel_l2
from parity_util import FIELDS9, TOL_1STEP, assert_particles_bitwise

pytestmark = pytest.mark.gpu


def _pair(cells, species, dtype, shape="tsc", super_cell=(8, 8, 4), deltas=(1.0, 1.0, 1.0)):
    from oracle.pic import OracleSim
    from paper_1606_02862_b200.pic import SimParams, Simulation
    p = SimParams(cells=cells, species=species, dtype=dtype, shape=shape, super_cell=super_cell,
                  dx=deltas[0], dy=deltas[1], dz=deltas[2])
    gpu = Simulation(p, validate=True)
    orc = OracleSim(p, validate=True, shape_order=p.shape_order, threads=2)
    return p, gpu, orc


def _load(p, gpu, orc, records):
    """records: list (per species) of dicts of global-cell particle arrays."""
    gpu.load_state(particles=records)
    for st, rec in zip(orc.stores, records):
        scx, scy, scz = st.super_cell
        gx, gy, _ = st.sc_grid
        cx, cy, cz = (np.asarray(rec[k]).astype(np.int64) for k in ("cx", "cy", "cz"))
        sc = cx // scx + gx * (cy // scy + gy * (cz // scz))
        o = np.argsort(sc, kind="stable")
        st.load_packed(sc[o], {k: np.asarray(v)[o] for k, v in rec.items()})


def _step_and_compare(p, gpu, orc, steps=2, tol=None):
    dt = np.dtype(p.dtype)
    tol = tol or TOL_1STEP[dt]
    for t in range(steps):
        if t:
            gpu.load_state(fields={n: getattr(orc.fields, n) for n in FIELDS9},
                           particles=[st.packed() for st in orc.stores])
        gpu.step()
        orc.step()
        for gs, os_ in zip(gpu.stores, orc.stores):
            assert_particles_bitwise(gs, os_)
        for n in FIELDS9:
            err = rel_l2(gpu.fields.numpy(n), getattr(orc.fields, n))
            assert err <= tol, (t, n, err)
        assert gpu.last_residual <= (1e-12 if dt == np.float64 else 1e-6)


def _rec(cells_xyz, offs, us, w, dtype):
    c = np.asarray(cells_xyz, dtype=np.int32)
    o = np.asarray(offs, dtype=dtype)
    u = np.asarray(us, dtype=dtype)
    return dict(cx=c[:, 0], cy=c[:, 1], cz=c[:, 2], ox=o[:, 0], oy=o[:, 1], oz=o[:, 2],
                ux=u[:, 0], uy=u[:, 1], uz=u[:, 2], w=np.full(len(c), w, dtype=dtype))


def _electron(w=1.0):
    from paper_1606_02862_b200.pic import Species
    return (Species("electron", -1.0, 1.0, w),)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_empty_store_steps(dtype):
    p, gpu, orc = _pair((16, 16, 8), _electron(), dtype)
    gpu.step()
    assert gpu.census() == 0
    for n in FIELDS9:
        assert float(np.abs(gpu.fields.numpy(n)).max()) == 0.0


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_single_fast_particle_crossing_faces(dtype):
    """One electron at u ~ 7 c moving diagonally across super-cell faces and
    the periodic boundary (largest CFL displacement)."""
    p, gpu, orc = _pair((16, 16, 8), _electron(0.5), dtype)
    rec = _rec([[15, 7, 7]], [[0.9, 0.99, 0.95]], [[4.0, 4.0, 4.0]], 0.5, dtype)
    _load(p, gpu, orc, [rec])
    _step_and_compare(p, gpu, orc, steps=3)


def test_offsets_exactly_zero_and_one_f32():
    """fp32 offsets of exactly 0.0 and 1.0 (1.0 arises from rounding in the
    reference's move and must be carried, not clamped)."""
    dtype = np.float32
    p, gpu, orc = _pair((16, 16, 8), _electron(0.25), dtype)
    cells, offs, us = [], [], []
    rng = np.random.default_rng(1)
    for i in range(64):
        cells.append([rng.integers(0, 16), rng.integers(0, 16), rng.integers(0, 8)])
        o = rng.choice([0.0, 1.0, np.float32(1.0) - np.float32(2.0 ** -24), 0.5], size=3)
        offs.append(o)
        us.append(rng.normal(0.0, 0.3, 3))
    _load(p, gpu, orc, [_rec(cells, offs, us, 0.25, dtype)])
    _step_and_compare(p, gpu, orc, steps=2)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_single_super_cell_per_axis_selfwrap(dtype):
    """cells == super cell along x and z: leaving through a face re-enters
    the same super cell (periodic self-wrap)."""
    from paper_1606_02862_b200.pic import default_species
    p, gpu, orc = _pair((8, 16, 4), default_species(2, 1.0), dtype)
    rng = np.random.default_rng(2)
    n = 300
    recs = []
    for s in range(2):
        c = np.stack([rng.integers(0, 8, n), rng.integers(0, 16, n), rng.integers(0, 4, n)], 1)
        recs.append(_rec(c, rng.random((n, 3)), rng.normal(0.0, 1.0, (n, 3)), 0.5, dtype))
    _load(p, gpu, orc, recs)
    _step_and_compare(p, gpu, orc, steps=3)


@pytest.mark.parametrize("shape", ["cic", "tsc", "pcs"])
def test_small_super_cell_anisotropic_f64(shape):
    """(4,4,4) super cells (64-thread CTAs, generic kernel instance),
    anisotropic cell sizes, every shape in float64."""
    from paper_1606_02862_b200.pic import default_species
    p, gpu, orc = _pair((8, 12, 8), default_species(2, 3.0), np.float64, shape=shape,
                        super_cell=(4, 4, 4), deltas=(0.7, 1.0, 1.3))
    rng = np.random.default_rng(3)
    n = 400
    recs = []
    for s in range(2):
        c = np.stack([rng.integers(0, 8, n), rng.integers(0, 12, n), rng.integers(0, 8, n)], 1)
        recs.append(_rec(c, rng.random((n, 3)), rng.normal(0.0, 0.5, (n, 3)), 0.5, np.float64))
    _load(p, gpu, orc, recs)
    _step_and_compare(p, gpu, orc, steps=3)


def test_one_particle_per_cell_dense_columns():
    from paper_1606_02862_b200.pic import SimParams, Species, init_khi
    from oracle.pic import oracle_init_khi
    p = SimParams(cells=(16, 16, 16), species=(Species("e", -1.0, 1.0, 1.0),),
                  particles_per_cell=1, dtype=np.float32, stream_velocity=0.0,
                  perturbation=0.0, thermal_u=0.2)
    gpu = init_khi(p, seed=8, validate=True)
    orc = oracle_init_khi(p, seed=8, validate=True, threads=2)
    _step_and_compare(p, gpu, orc, steps=2)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_graph_replay_matches_direct_launches(dtype):
    """enqueue_step replays a captured CUDA graph (validate=False).  Teacher
    forced against direct launches: before every step of the graph-driven
    simulation its state is loaded into a directly launched one; one step
    later the particle state is bitwise equal and the fields agree to the
    rounding of the J atomics."""
    import torch
    from paper_1606_02862_b200.pic import SimParams, default_species, init_khi
    p = SimParams(cells=(16, 16, 8), species=default_species(4, 4.0), particles_per_cell=4,
                  dtype=dtype, thermal_u=0.3)
    a = init_khi(p, seed=3, validate=False)
    b = init_khi(p, seed=3, validate=False)
    a.use_graphs, b.use_graphs = True, False
    a.enqueue_step()
    b.enqueue_step()
    tol = TOL_1STEP[np.dtype(dtype)]
    for t in range(4):
        b.load_state(fields={n: a.fields.numpy(n) for n in FIELDS9},
                     particles=[st.packed() for st in a.stores])
        a.enqueue_step()
        b.enqueue_step()
        a.check_status()
        b.check_status()
        torch.cuda.synchronize()
        for sa, sb in zip(a.stores, b.stores):
            assert_particles_bitwise(sa, sb)
        for n in FIELDS9:
            assert rel_l2(a.fields.numpy(n), b.fields.numpy(n)) <= tol, (t, n)
    assert len(a._graphs) == 2 and not b._graphs   # one graph per buffer parity, replayed


def _records_sorted(pk):
    from parity_util import sorted_records
    return sorted_records(pk)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_clumped_load_retries_with_larger_columns(dtype):
    """Columns are first sized from the mean load; 3000 particles in one cell
    overflow that, and the load is redone from the fullest cell's count."""
    import torch
    from paper_1606_02862_b200.pic import SimParams, Species, Simulation
    p = SimParams(cells=(16, 16, 8), species=(Species("e", -1.0, 1.0, 1.0),), dtype=dtype)
    sim = Simulation(p, validate=False)
    rng = np.random.default_rng(0)
    n = 3000
    cells = np.tile([[5, 6, 3]], (n, 1))
    rec = _rec(cells, rng.random((n, 3)), rng.normal(0, 0.1, (n, 3)), 1.0, dtype)
    rec["cx"][:10] = 0   # a few elsewhere
    sim.load_state(particles=[rec])
    st = sim.stores[0]
    assert st.frames_per_sc >= n - 10
    assert st.census() == n and st.check_integrity()
    got, want = _records_sorted(st.packed()), _records_sorted(rec)
    for k in want:
        np.testing.assert_array_equal(got[k], want[k])
    torch.cuda.synchronize()


@pytest.mark.parametrize("aligned", [True, False])
def test_column_range_export_with_clear(aligned):
    """packed_device over a column range (whole super cells: the staged
    export; a ragged range: the per-column export) returns exactly those
    columns' particles in canonical order and empties them when asked."""
    from paper_1606_02862_b200.pic import SimParams, default_species, init_khi
    p = SimParams(cells=(16, 16, 8), species=default_species(4, 1.0), particles_per_cell=4,
                  dtype=np.float32, thermal_u=0.2)
    sim = init_khi(p, seed=1, validate=False)
    for _ in range(2):
        sim.step()
    st = sim.stores[0]
    V = st.capacity
    c0, c1 = (V, 3 * V) if aligned else (V + 7, 3 * V - 5)
    full = st.packed()
    # expected: records of those columns, canonical (super cell, cell, frame) order
    scx, scy, scz = st.super_cell
    gx, gy, _ = st.sc_grid
    sc = full["cx"] // scx + gx * (full["cy"] // scy + gy * (full["cz"] // scz))
    lc = (full["cx"] % scx) + scx * ((full["cy"] % scy) + scy * (full["cz"] % scz))
    col = sc.astype(np.int64) * V + lc
    m = (col >= c0) & (col < c1)
    part = {k: v.cpu().numpy() for k, v in st.packed_device(columns=(c0, c1), clear=True).items()}
    assert part["cx"].shape[0] == int(m.sum())
    pc = (part["cx"] // scx + gx * (part["cy"] // scy + gy * (part["cz"] // scz))).astype(np.int64) * V \
        + (part["cx"] % scx) + scx * ((part["cy"] % scy) + scy * (part["cz"] % scz))
    assert np.all(np.diff(pc) >= 0)   # column-major (canonical) order
    got, want = _records_sorted(part), _records_sorted({k: v[m] for k, v in full.items()})
    for k in want:
        np.testing.assert_array_equal(got[k], want[k])
    rest = st.packed()
    assert rest["cx"].shape[0] == full["cx"].shape[0] - int(m.sum())
    assert st.check_integrity()


@pytest.mark.parametrize("dtype,shape", [(np.float32, "cic"), (np.float32, "tsc"),
                                         (np.float64, "tsc"), (np.float32, "pcs")])
def test_zslab_entry_identity_plane_table_matches_advance(dtype, shape):
    """kwb_particles_advance_zslab with the identity plane table (every J
    plane z of component c -> plane z of J[c]) is kwb_particles_advance:
    particles bitwise, fields to the rounding of the J atomics; a table that
    routes every plane into a second J buffer leaves J itself zero and
    deposits the same current there."""
    import torch
    from paper_1606_02862_b200.pic import SimParams, default_species, init_khi
    p = SimParams(cells=(16, 16, 8), species=default_species(4, 4.0), particles_per_cell=4,
                  dtype=dtype, thermal_u=0.3, shape=shape)
    a = init_khi(p, seed=5, validate=False)
    b = init_khi(p, seed=5, validate=False)
    a.use_graphs = b.use_graphs = False
    nz = p.cells.as_tuple()[2]
    J3 = ("Jx", "Jy", "Jz")
    b._jplanes = torch.tensor([b.fields.storage(n)[z].data_ptr() for n in J3 for z in range(nz)],
                              dtype=torch.int64, device=b.device)
    tol = TOL_1STEP[np.dtype(dtype)]
    for t in range(2):
        # teacher forced: the J atomics' summation order differs between
        # runs, so each step starts b from a's state
        b.load_state(fields={n: a.fields.numpy(n) for n in FIELDS9},
                     particles=[st.packed() for st in a.stores])
        a.enqueue_step()
        b.enqueue_step()
        a.check_status()
        b.check_status()
        for sa, sb in zip(a.stores, b.stores):
            assert_particles_bitwise(sa, sb)
        for n in FIELDS9:
            assert rel_l2(b.fields.numpy(n), a.fields.numpy(n)) <= tol, (t, n)
    b.load_state(fields={n: a.fields.numpy(n) for n in FIELDS9},
                 particles=[st.packed() for st in a.stores])
    # redirect every plane into a side buffer: J stays zero, the side holds it
    side = torch.zeros((3,) + tuple(b.fields.storage("Jx").shape), dtype=b.fields.storage("Jx").dtype,
                       device=b.device)
    b._jplanes = torch.tensor([side[c][z].data_ptr() for c in range(3) for z in range(nz)],
                              dtype=torch.int64, device=b.device)
    a.advance_particles()
    b.advance_particles()
    torch.cuda.synchronize()
    for c, n in enumerate(J3):
        assert float(b.fields.storage(n).abs().max()) == 0.0
        want = a.fields.storage(n).double().cpu().numpy()
        assert rel_l2(side[c].double().cpu().numpy(), want) <= tol, n
