"""z-slab decomposition on the CUDA path, verified on ONE GPU: G virtual
ranks (LoopbackTransport: exchanges are copies between the ranks' buffers, so
no kernel ever waits on another rank) against the single-domain CUDA run.
The multi-process NCCL transport shares every line of this logic except
DistTransport, which tests/test_decomp_cpu.py covers with gloo."""

import numpy as np
import pytest

from golden_util import rel_l2

pytestmark = pytest.mark.gpu

FIELDS9 = ("Ex", "Ey", "Ez", "Bx", "By", "Bz", "Jx", "Jy", "Jz")
PK = ("cx", "cy", "cz", "ox", "oy", "oz", "ux", "uy", "uz", "w")


def _sorted(pk):
    keys = []
    for k in reversed(PK):
        a = np.asarray(pk[k])
        keys.append(a.view(np.uint64 if a.itemsize == 8 else np.uint32) if a.dtype.kind == "f" else a)
    o = np.lexsort(keys)
    return {k: np.asarray(pk[k])[o] for k in PK}


@pytest.mark.parametrize("fuse_j", [False, True])
@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("dtype,shape", [(np.float64, "tsc"), (np.float32, "tsc"), (np.float32, "pcs")])
def test_loopback_slabs_match_single_domain(world, dtype, shape, fuse_j):
    """fuse_j=True: guard-plane J deposited straight into the owning slab's
    planes (kwb_particles_advance_zslab), no J exchange; False: the
    exchanged-and-summed guard planes the multi-process path uses."""
    from paper_1606_02862_b200.pic import SimParams, default_species, init_khi
    from paper_1606_02862_b200.pic.decomp import DecomposedSimulation, LoopbackTransport
    p = SimParams(cells=(16, 16, 24), species=default_species(4, 4.0), particles_per_cell=4,
                  dtype=np.dtype(dtype), stream_velocity=0.2, perturbation=0.05, thermal_u=0.1,
                  shape=shape)
    ref = init_khi(p, seed=9, validate=False)
    dec = DecomposedSimulation(p, world, range(world), LoopbackTransport(), fuse_j=fuse_j)
    assert dec.fuse_j == fuse_j
    dec.load_global(particles=[st.packed() for st in ref.stores])
    dec.refresh_guards()
    n0 = ref.census()
    tol = 1e-13 if np.dtype(dtype) == np.float64 else 1e-5
    for t in range(3):
        ref.step()
        dec.step()
        dec.check_status()
        assert dec.census() == n0
        for i in range(len(p.species)):
            full = ref.stores[i].packed()
            mine = _sorted({k: np.concatenate([dec.owned_particles(r, i)[k] for r in range(world)])
                            for k in PK})
            want = _sorted(full)
            for k in ("cx", "cy", "cz"):
                np.testing.assert_array_equal(mine[k], want[k], err_msg=f"step {t} {k}")
            for k in ("ox", "oy", "oz", "ux", "uy", "uz", "w"):
                if t == 0:
                    np.testing.assert_array_equal(mine[k], want[k], err_msg=k)
                else:
                    np.testing.assert_allclose(mine[k], want[k], rtol=100 * tol, atol=10 * tol)
        for n in FIELDS9:
            got = np.concatenate([dec.owned_fields(r, n) for r in range(world)], axis=2)
            err = rel_l2(got, ref.fields.numpy(n))
            assert err <= tol * (1 + 10 * t), (t, n, err)


def test_decomposed_diagnostics_match_single_domain():
    from paper_1606_02862_b200.pic import SimParams, default_species, init_khi
    from paper_1606_02862_b200.pic.decomp import DecomposedSimulation, LoopbackTransport
    p = SimParams(cells=(16, 16, 24), species=default_species(4, 4.0), particles_per_cell=4,
                  dtype=np.float64, stream_velocity=0.2, perturbation=0.05, thermal_u=0.1)
    ref = init_khi(p, seed=9, validate=False)
    dec = DecomposedSimulation(p, 3, range(3), LoopbackTransport())
    dec.load_global(particles=[st.packed() for st in ref.stores])
    dec.refresh_guards()
    for _ in range(3):
        ref.step()
        dec.step()
    a, b = dec.diagnostics(), ref.diagnostics()
    assert a["total_charge"] == pytest.approx(b["total_charge"], rel=1e-12, abs=1e-12)
    assert a["kinetic_energy"] == pytest.approx(b["kinetic_energy"], rel=1e-12)
    assert a["field_energy"] == pytest.approx(b["field_energy"], rel=1e-9)
    assert a["max_div_b"] <= 1e-12 and b["max_div_b"] <= 1e-12


def _fast_pair(world):
    from paper_1606_02862_b200.pic import SimParams, default_species, init_khi
    from paper_1606_02862_b200.pic.decomp import DecomposedSimulation, LoopbackTransport
    p = SimParams(cells=(16, 16, 24), species=default_species(4, 4.0), particles_per_cell=4,
                  dtype=np.float64, stream_velocity=0.0, perturbation=0.0, thermal_u=1.0)
    ref = init_khi(p, seed=5, validate=False)
    dec = DecomposedSimulation(p, world, range(world), LoopbackTransport())
    dec.load_global(particles=[st.packed() for st in ref.stores])
    dec.refresh_guards()
    return p, ref, dec


def test_guard_exchange_overflow_is_redone():
    """Fixed-capacity guard messages far too small for a hot plasma: the
    checked step detects the overflow, doubles the messages and redoes the
    exchange -- the result equals the single-domain run, nothing is lost."""
    p, ref, dec = _fast_pair(2)
    dec._xcap = 2
    n0 = ref.census()
    for _ in range(2):
        ref.step()
        dec.step()
        dec.check_status()
        assert dec.census() == n0
    assert dec._xcap > 2
    for i in range(len(p.species)):
        mine = _sorted({k: np.concatenate([dec.owned_particles(r, i)[k] for r in range(2)])
                        for k in PK})
        want = _sorted(ref.stores[i].packed())
        for k in ("cx", "cy", "cz"):
            np.testing.assert_array_equal(mine[k], want[k])


def test_guard_exchange_overflow_raises_when_unchecked():
    from paper_1606_02862_b200.errors import AllocationError
    p, ref, dec = _fast_pair(2)
    dec._xcap = 2
    with pytest.raises(AllocationError, match="guard-layer"):
        for _ in range(3):
            dec.enqueue_step()
        dec.check_status()


def test_decomposed_checked_step_raises_before_field_update():
    """checked step (the reference's synchronous semantics across slabs): a
    particle that moves a full cell raises ContractViolation right after
    the advance, before any exchange or field update (E and B untouched)."""
    from paper_1606_02862_b200.errors import ContractViolation
    from paper_1606_02862_b200.pic import SimParams, Species
    from paper_1606_02862_b200.pic.decomp import DecomposedSimulation, LoopbackTransport
    p = SimParams(cells=(16, 16, 24), species=(Species("e", -1.0, 1.0, 1.0),), dtype=np.float64)
    dec = DecomposedSimulation(p, 2, range(2), LoopbackTransport())
    pk = dict(cx=np.array([3, 5]), cy=np.array([3, 5]), cz=np.array([1, 14]),
              ox=np.array([0.5, 3.0]), oy=np.array([0.5, 0.5]), oz=np.array([0.5, 0.5]),
              ux=np.zeros(2), uy=np.zeros(2), uz=np.zeros(2), w=np.ones(2))
    ex = np.full((16, 16, 24), 0.125)
    dec.load_global(fields={"Ex": ex}, particles=[pk])
    dec.refresh_guards()
    with pytest.raises(ContractViolation, match="1 particle"):
        dec.step()
    got = np.concatenate([dec.owned_fields(r, "Ex") for r in range(2)], axis=2)
    np.testing.assert_array_equal(got, ex)
    assert np.isnan(dec.diagnostics()["max_continuity_residual"])
