"""CUDA path vs the pinned oracle and the reference's golden dumps (B200).

Bars (north_star):
* particle records (cells, offsets, momenta, weights) and super-cell
  membership BITWISE after one step from identical state, any dtype;
* J/E/B within relative L2 1e-13 (f64) / 1e-6 (f32) after one step and
  1e-12 / 1e-4 free-running;
* census exact, per-cell occupancy exact (f64) or <= 4 displaced (f32);
* continuity residual and Gauss drift within 1e-12 / 1e-6 every step.
"""

import numpy as np
import pytest
import torch

from golden_util import CASES, load_case, oracle_params, rel_l2
from parity_util import (FIELDS9, TOL_1STEP, TOL_FREE, TOL_GAUSS, TOL_RESID,
                         assert_particles_bitwise, check_fields, order_spread, gpu_params, make_pair,
                         occupancy, record)

pytestmark = pytest.mark.gpu


def _dtype(meta):
    return np.dtype(meta["config"]["dtype"])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("deltas", [(1.0, 1.0, 1.0), (0.7, 1.0, 1.3)])
def test_yee_update_bitwise(dtype, deltas):
    """Faraday-Ampere-Faraday on random E/B/J equals the oracle bit for bit."""
    from oracle.pic import OracleFields, lib as olib
    from paper_1606_02862_b200.pic import SimParams, Simulation, Species
    import ctypes
    cells = (16, 24, 12)
    p = SimParams(cells=cells, dx=deltas[0], dy=deltas[1], dz=deltas[2],
                  species=(Species("e", -1.0, 1.0, 1.0),), super_cell=(8, 8, 4), dtype=dtype)
    sim = Simulation(p, validate=False)
    of = OracleFields(cells, *deltas, dtype)
    rng = np.random.default_rng(5)
    for n in FIELDS9:
        a = rng.standard_normal(cells).astype(dtype)
        setattr(of, n, a)
        sim.fields.load_numpy(n, a)
    sim.update_fields()
    cf = of._cfields()
    sfx = "_f32" if np.dtype(dtype) == np.float32 else "_f64"
    getattr(olib(), "orc_faraday" + sfx)(ctypes.byref(cf), p.dt / 2.0, 4)
    getattr(olib(), "orc_ampere" + sfx)(ctypes.byref(cf), p.dt, 4)
    getattr(olib(), "orc_faraday" + sfx)(ctypes.byref(cf), p.dt / 2.0, 4)
    for n in FIELDS9:
        np.testing.assert_array_equal(sim.fields.numpy(n), getattr(of, n), err_msg=n)


@pytest.mark.parametrize("name", CASES)
def test_one_step_vs_oracle(name):
    meta, _ = load_case(name)
    gpu, orc = make_pair(meta)
    for gs, os_ in zip(gpu.stores, orc.stores):
        assert_particles_bitwise(gs, os_)            # identical initial state
    spread = order_spread(orc)
    gpu.step()
    orc.step()
    for gs, os_ in zip(gpu.stores, orc.stores):
        assert_particles_bitwise(gs, os_)
    check_fields(f"{name}:init", gpu.fields, lambda n: getattr(orc.fields, n),
                 TOL_1STEP[_dtype(meta)], spread=spread)
    assert gpu.last_residual <= TOL_RESID[_dtype(meta)]


@pytest.mark.parametrize("name", CASES)
def test_teacher_forced_from_evolved_state(name):
    """Load the oracle's state after 3 steps (non-zero fields, migrated
    particles) into the GPU, step both once, compare bitwise."""
    meta, _ = load_case(name)
    gpu, orc = make_pair(meta, validate=False)
    orc.run(3)
    gpu.load_state(fields={n: getattr(orc.fields, n) for n in FIELDS9},
                   particles=[st.packed() for st in orc.stores])
    for gs, os_ in zip(gpu.stores, orc.stores):
        assert_particles_bitwise(gs, os_)
    spread = order_spread(orc)
    gpu.step()
    orc.step()
    for gs, os_ in zip(gpu.stores, orc.stores):
        assert_particles_bitwise(gs, os_)
    check_fields(f"{name}:evolved3", gpu.fields, lambda n: getattr(orc.fields, n),
                 TOL_1STEP[_dtype(meta)], spread=spread)


@pytest.mark.parametrize("name", CASES)
def test_free_running_vs_reference_golden(name):
    """Free-running from init against the reference's own dumps."""
    meta, data = load_case(name)
    from paper_1606_02862_b200.pic import init_khi
    op = oracle_params(meta)
    sim = init_khi(gpu_params(op), seed=meta["config"]["seed"], validate=True)
    dt = _dtype(meta)
    steps = sorted(int(k[1:]) for k in meta["steps"])
    for t in range(max(steps) + 1):
        if t in steps:
            key = f"t{t}"
            sm = meta["steps"][key]
            assert sim.census() == sm["census"]
            for i, st in enumerate(sim.stores):
                occ = occupancy(st.packed(), op.cells)
                ref = data[f"{key}_s{i}_occupancy"].astype(np.int64)
                displaced = int(np.abs(occ - ref).sum()) // 2
                assert displaced <= (0 if dt == np.float64 else 4), (key, i, displaced)
            check_fields(f"{name}:free:{key}", sim.fields, lambda n: data[f"{key}_{n}"],
                         TOL_FREE[dt], kind="free")
            if t > 0:
                assert sim.last_residual <= TOL_RESID[dt]
                assert sim.last_gauss_drift <= TOL_GAUSS[dt]
                d = sim.diagnostics()
                ref_d = sm["diagnostics"]
                assert d["total_charge"] == pytest.approx(ref_d["total_charge"], rel=1e-9, abs=1e-12)
                assert d["kinetic_energy"] == pytest.approx(ref_d["kinetic_energy"], rel=1e-6)
                assert d["field_energy"] == pytest.approx(ref_d["field_energy"], rel=1e-3, abs=1e-12)
        if t < max(steps):
            sim.step()


@pytest.mark.parametrize("shape", ["cic", "pcs"])
@pytest.mark.parametrize("name", ["thermal_e_f64", "eion_f32"])
def test_extended_shapes_vs_oracle(shape, name):
    """CIC and PCS (SURVEY.md §8c extension): teacher-forced steps give
    bitwise particles and J within tolerance of the extended oracle; charge
    is conserved per step (continuity and Gauss drift)."""
    meta, _ = load_case(name)
    gpu, orc = make_pair(meta, shape=shape)
    dt = _dtype(meta)
    for it in range(3):
        if it:
            gpu.load_state(fields={n: getattr(orc.fields, n) for n in FIELDS9},
                           particles=[st.packed() for st in orc.stores])
        spread = order_spread(orc)
        gpu.step()
        orc.step()
        for gs, os_ in zip(gpu.stores, orc.stores):
            assert_particles_bitwise(gs, os_)
        check_fields(f"{name}:{shape}:step{it}", gpu.fields, lambda n: getattr(orc.fields, n),
                     TOL_1STEP[dt], spread=spread)
        assert gpu.last_residual <= TOL_RESID[dt]
        assert orc.last_residual <= TOL_RESID[dt]
        if it == 0:
            assert gpu.last_gauss_drift <= TOL_GAUSS[dt]


def test_contract_violation_on_full_cell_move():
    from paper_1606_02862_b200.errors import ContractViolation
    from paper_1606_02862_b200.pic import SimParams, Simulation, Species
    p = SimParams(cells=(16, 16, 8), species=(Species("e", -1.0, 1.0, 1.0),),
                  dtype=np.float64)
    sim = Simulation(p, validate=False)
    pk = dict(cx=np.array([3, 5]), cy=np.array([3, 5]), cz=np.array([1, 2]),
              ox=np.array([0.5, 3.0]), oy=np.array([0.5, 0.5]), oz=np.array([0.5, 0.5]),
              ux=np.zeros(2), uy=np.zeros(2), uz=np.zeros(2), w=np.ones(2))
    sim.load_state(particles=[pk])
    with pytest.raises(ContractViolation, match="1 particle"):
        sim.step()


def test_stationary_particle_gives_zero_current_and_uniform_field_gather():
    """SPEC KATs: stationary particle -> J = 0; uniform E -> u' = u + q dt E/m
    (dyadic offsets keep the trilinear weights exact)."""
    from paper_1606_02862_b200.pic import SimParams, Simulation, Species
    p = SimParams(cells=(16, 16, 8), species=(Species("e", -1.0, 1.0, 0.5),),
                  dtype=np.float64)
    sim = Simulation(p, validate=False)
    rng = np.random.default_rng(3)
    n = 500
    pk = dict(cx=rng.integers(0, 16, n), cy=rng.integers(0, 16, n), cz=rng.integers(0, 8, n),
              ox=rng.integers(0, 8, n) / 8.0, oy=rng.integers(0, 8, n) / 8.0,
              oz=rng.integers(0, 8, n) / 8.0,
              ux=np.zeros(n), uy=np.zeros(n), uz=np.zeros(n), w=np.full(n, 0.5))
    sim.load_state(particles=[pk])
    sim.step()
    for n_ in ("Jx", "Jy", "Jz"):
        assert float(sim.fields.numpy(n_).__abs__().max()) == 0.0
    # uniform Ex: gathered exactly, B = 0 => u = 2 * qm * Ex exactly (double)
    sim2 = Simulation(p, validate=False)
    ex = np.full((16, 16, 8), 0.25)
    sim2.load_state(fields={"Ex": ex}, particles=[pk])
    sim2.enqueue_step()
    out = sim2.stores[0].packed()
    qm = -1.0 * p.dt / 2.0
    expect = (0.0 + qm * 0.25) + qm * 0.25
    np.testing.assert_array_equal(out["ux"], np.full(n, expect))


def test_store_growth_keeps_particles():
    """Force a capacity repack mid-run: census and state survive."""
    meta, _ = load_case("eion_f32")
    gpu, orc = make_pair(meta, validate=False)
    st = gpu.stores[0]
    before = st.packed()
    st.reserve(st.frames_per_sc)   # > 85% of the frames -> grow
    assert st.check_integrity()
    after = st.packed()
    for k in before:
        np.testing.assert_array_equal(np.sort(before[k]), np.sort(after[k]))
    gpu.step()
    orc.step()
    for gs, os_ in zip(gpu.stores, orc.stores):
        assert_particles_bitwise(gs, os_)


def test_store_api_surface():
    from paper_1606_02862_b200.pic import MacroParticle
    meta, _ = load_case("thermal_e_f64")
    gpu, orc = make_pair(meta, validate=False)
    st = gpu.stores[0]
    assert st.census() == orc.stores[0].census()
    assert st.check_integrity()
    assert int(st.occ.sum()) == st.census()
    assert int(st.nfilled.sum()) == st.census()
    assert st.frames_of(0) == [0, 1, 2, 3, 4, 5, 6, 7][: len(st.frames_of(0))]
    parts = list(st.iter_particles())
    assert len(parts) == st.census()
    st.insert(MacroParticle((1, 2, 3), (0.25, 0.5, 0.75), (0.1, 0.0, 0.0), 0.125))
    assert st.census() == orc.stores[0].census() + 1
    assert st.check_integrity()


@pytest.mark.slow
def test_c2_shape_properties_at_64cubed():
    """C2's species mix and distribution at 64^3: census conserved, charge
    conserved (continuity and Gauss drift) every step in fp32."""
    from paper_1606_02862_b200.pic import SimParams, default_species, init_khi
    p = SimParams(cells=(64, 64, 64), species=default_species(25, 1836.0),
                  particles_per_cell=25, dtype=np.float32, stream_velocity=0.0,
                  perturbation=0.0, thermal_u=0.05)
    sim = init_khi(p, seed=2, validate=True)
    n0 = sim.census()
    assert n0 == 64 ** 3 * 25 * 2
    for _ in range(5):
        sim.step()
        assert sim.census() == n0
        assert sim.last_residual <= 1e-6
        assert sim.last_gauss_drift <= 1e-6
    for st in sim.stores:
        assert st.check_integrity()
    torch.cuda.synchronize()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_field_helpers_gather_and_yee(dtype):
    """Module helpers of the reference's pic/fields.py: yee_update_b /
    yee_update_e equal the oracle's Faraday / Ampere bit for bit, and
    gather_fields equals the reference's trilinear recipe (pic/kernels.py
    :26-47, double arithmetic, rounded to the storage type) at random
    points, bit for bit."""
    from oracle.pic import OracleFields, lib as olib
    import ctypes
    from paper_1606_02862_b200.pic import (MacroParticle, STAGGER, YeeFieldSet, gather_fields,
                                           yee_update_b, yee_update_e)
    cells = (12, 10, 8)
    deltas = (0.7, 1.0, 1.3)
    f = YeeFieldSet(cells, *deltas, dtype=dtype)
    of = OracleFields(cells, *deltas, dtype)
    rng = np.random.default_rng(17)
    for n in FIELDS9:
        a = rng.standard_normal(cells).astype(dtype)
        setattr(of, n, a)
        f.load_numpy(n, a)
    dt = 0.4
    yee_update_b(f, dt / 2.0)
    yee_update_e(f, dt)
    cf = of._cfields()
    sfx = "_f32" if np.dtype(dtype) == np.float32 else "_f64"
    getattr(olib(), "orc_faraday" + sfx)(ctypes.byref(cf), dt / 2.0, 2)
    getattr(olib(), "orc_ampere" + sfx)(ctypes.byref(cf), dt, 2)
    for n in FIELDS9:
        np.testing.assert_array_equal(f.numpy(n), getattr(of, n), err_msg=n)

    def sample(a, px, py, pz, s):
        nx, ny, nz = a.shape
        tx, ty, tz = px - s[0], py - s[1], pz - s[2]
        ix, iy, iz = int(np.floor(tx)), int(np.floor(ty)), int(np.floor(tz))
        fx, fy, fz = tx - ix, ty - iy, tz - iz
        A = lambda i, j, k: float(a[i % nx, j % ny, k % nz])
        c00 = A(ix, iy, iz) * (1.0 - fx) + A(ix + 1, iy, iz) * fx
        c10 = A(ix, iy + 1, iz) * (1.0 - fx) + A(ix + 1, iy + 1, iz) * fx
        c01 = A(ix, iy, iz + 1) * (1.0 - fx) + A(ix + 1, iy, iz + 1) * fx
        c11 = A(ix, iy + 1, iz + 1) * (1.0 - fx) + A(ix + 1, iy + 1, iz + 1) * fx
        return (c00 * (1.0 - fy) + c10 * fy) * (1.0 - fz) + (c01 * (1.0 - fy) + c11 * fy) * fz

    ps = [MacroParticle((int(rng.integers(0, cells[0])), int(rng.integers(0, cells[1])),
                         int(rng.integers(0, cells[2]))),
                        tuple(float(np.asarray(x, dtype=dtype)) for x in rng.random(3)),
                        (0.0, 0.0, 0.0)) for _ in range(200)]
    ps.append(MacroParticle((0, 0, 0), (0.0, 1.0, 0.5), (0.0, 0.0, 0.0)))
    e, b = gather_fields(f, ps)
    for q, p in enumerate(ps):
        px, py, pz = (p.cell[a] + p.offset[a] for a in range(3))
        want = [np.asarray(sample(f.numpy(n), px, py, pz, STAGGER[n]), dtype=dtype)
                for n in ("Ex", "Ey", "Ez", "Bx", "By", "Bz")]
        got = list(e[q]) + list(b[q])
        for w_, g_ in zip(want, got):
            assert np.asarray(g_, dtype=dtype).tobytes() == w_.tobytes()
    e1, b1 = gather_fields(f, ps[0])
    assert e1.shape == (3,) and b1.shape == (3,)


@pytest.mark.parametrize("mode", ["fused", "per_species_calls", "shared_exchange"])
def test_species_paths_agree_with_oracle(mode, monkeypatch):
    """The three particle-phase paths: two species in one fused launch
    (KWB_SPECIES_FUSION=1), the reference's per-species advance + shift
    calls (KWB_PER_SPECIES=1), and per-species launches sharing one
    exchange buffer with one shift for all species (default).  Teacher
    forced from the oracle's evolved state of a hot e/ion plasma: particles
    bitwise, fields within the bars."""
    monkeypatch.setenv("KWB_SPECIES_FUSION", "1" if mode == "fused" else "0")
    monkeypatch.setenv("KWB_PER_SPECIES", "1" if mode == "per_species_calls" else "0")
    meta, _ = load_case("eion_f32")
    gpu, orc = make_pair(meta, validate=False)
    assert gpu.fuse_species == (mode != "per_species_calls")
    orc.run(2)
    gpu.load_state(fields={n: getattr(orc.fields, n) for n in FIELDS9},
                   particles=[st.packed() for st in orc.stores])
    spread = order_spread(orc)
    gpu.step()
    orc.step()
    for gs, os_ in zip(gpu.stores, orc.stores):
        assert_particles_bitwise(gs, os_)
    check_fields(f"eion_f32:{mode}", gpu.fields, lambda n: getattr(orc.fields, n),
                 TOL_1STEP[np.dtype(np.float32)], spread=spread)


def test_three_species_share_one_exchange_buffer():
    """Three species (more than the fused launch takes): one advance launch
    per species into ONE exchange buffer (dest = super cell + species x
    n_super_cells) and one shift launch that returns every leaver to its own
    species' store -- against the oracle, hot plasma (many leavers)."""
    from oracle.pic import OracleSim
    from paper_1606_02862_b200.pic import SimParams, Simulation, Species
    sp = (Species("e", -1.0, 1.0, 0.25), Species("p", 1.0, 4.0, 0.25), Species("x", -2.0, 9.0, 0.5))
    p = SimParams(cells=(16, 16, 8), species=sp, dtype=np.float32)
    gpu = Simulation(p, validate=True)
    orc = OracleSim(p, validate=True, shape_order=2, threads=2)
    rng = np.random.default_rng(41)
    recs = []
    for _ in sp:
        n = 3000
        recs.append(dict(cx=rng.integers(0, 16, n).astype(np.int32), cy=rng.integers(0, 16, n).astype(np.int32),
                         cz=rng.integers(0, 8, n).astype(np.int32),
                         ox=rng.random(n).astype(np.float32), oy=rng.random(n).astype(np.float32),
                         oz=rng.random(n).astype(np.float32),
                         ux=(0.6 * rng.standard_normal(n)).astype(np.float32),
                         uy=(0.6 * rng.standard_normal(n)).astype(np.float32),
                         uz=(0.6 * rng.standard_normal(n)).astype(np.float32),
                         w=np.full(n, 0.25, np.float32)))
    gpu.load_state(particles=recs)
    for st, rec in zip(orc.stores, recs):
        scx, scy, scz = st.super_cell
        gx, gy, _ = st.sc_grid
        scid = rec["cx"] // scx + gx * (rec["cy"] // scy + gy * (rec["cz"] // scz))
        o = np.argsort(scid, kind="stable")
        st.load_packed(scid[o], {k: np.asarray(v)[o] for k, v in rec.items()})
    spread = order_spread(orc)
    gpu.step()
    orc.step()
    for gs, os_ in zip(gpu.stores, orc.stores):
        assert_particles_bitwise(gs, os_)
    check_fields("three_species", gpu.fields, lambda n: getattr(orc.fields, n),
                 TOL_1STEP[np.dtype(np.float32)], spread=spread)
    assert gpu.last_residual <= TOL_RESID[np.dtype(np.float32)]


def test_multi_gpu_plumbing_on_one_device():
    """kwb_enable_peer_access to the own device is a no-op success and
    kwb_copy_async copies on the caller's stream (the z-slab plane pulls)."""
    from paper_1606_02862_b200 import _lib
    _lib.load()
    _lib.call("kwb_enable_peer_access", torch.cuda.current_device())
    a = torch.arange(4096, dtype=torch.float32, device="cuda")
    b = torch.zeros_like(a)
    _lib.call("kwb_copy_async", b.data_ptr(), a.data_ptr(), a.numel() * 4,
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
