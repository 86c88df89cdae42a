"""z-slab decomposition host logic on CPU: world-size 2 (and 3) gloo runs of
DecomposedSimulation with oracle-backed slabs, against a single-domain oracle
run.  Exercises the J-halo sum, guard-layer particle extraction/append with
global<->local z translation, the E/B guard exchanges and the message pairing
of DistTransport (lower == upper neighbour when G = 2)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_util import rel_l2

FIELDS9 = ("Ex", "Ey", "Ez", "Bx", "By", "Bz", "Jx", "Jy", "Jz")
PK = ("cx", "cy", "cz", "ox", "oy", "oz", "ux", "uy", "uz", "w")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _params(dtype, two_species):
    from paper_1606_02862_b200.pic import SimParams, Species, default_species
    sp = default_species(4, 1.0) if two_species else (Species("electron", -1.0, 1.0, 0.25),)
    return SimParams(cells=(16, 8, 24), species=sp, particles_per_cell=4,
                     dtype=np.dtype(dtype), stream_velocity=0.2, perturbation=0.05,
                     thermal_u=0.1, super_cell=(8, 8, 4))


def _sorted(pk):
    keys = []
    for k in reversed(PK):
        a = np.asarray(pk[k])
        keys.append(a.view(np.uint64 if a.itemsize == 8 else np.uint32) if a.dtype.kind == "f" else a)
    o = np.lexsort(keys)
    return {k: np.asarray(pk[k])[o] for k in PK}


def _worker(rank, world, port, dtype, two_species, steps):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pic import oracle_init_khi
        from oracle_slab import OracleLocal
        from paper_1606_02862_b200.pic.decomp import DecomposedSimulation, DistTransport
        p = _params(dtype, two_species)
        ref = oracle_init_khi(p, seed=5, validate=False, threads=2)
        dec = DecomposedSimulation(p, world, [rank], DistTransport(), local_factory=OracleLocal)
        dec.load_global(particles=[st.packed() for st in ref.stores])
        dec.refresh_guards()
        lay = dec.layouts[rank]
        n0 = ref.census()
        assert dec.census() == n0
        tol = 1e-13 if np.dtype(dtype) == np.float64 else 1e-5
        for t in range(steps):
            ref.step()
            dec.step()
            assert dec.census() == n0, "census not conserved across slabs"
            for i, st in enumerate(ref.stores):
                full = st.packed()
                m = (full["cz"] >= lay.z0) & (full["cz"] < lay.z0 + lay.nzl)
                mine = _sorted(dec.owned_particles(rank, i))
                want = _sorted({k: v[m] for k, v in full.items()})
                for k in ("cx", "cy", "cz"):
                    np.testing.assert_array_equal(mine[k], want[k], err_msg=f"step {t} {k}")
                for k in ("ox", "oy", "oz", "ux", "uy", "uz", "w"):
                    if t == 0:   # identical inputs -> bitwise
                        np.testing.assert_array_equal(mine[k], want[k], err_msg=f"{k}")
                    else:        # fields differ at rounding level after the halo sum
                        np.testing.assert_allclose(mine[k], want[k], rtol=100 * tol, atol=10 * tol)
            for n in FIELDS9:
                a = dec.owned_fields(rank, n)
                b = getattr(ref.fields, n)[:, :, lay.z0:lay.z0 + lay.nzl]
                assert rel_l2(a, b) <= tol * (1 + 10 * t), (t, n, rel_l2(a, b))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dtype,two", [(2, np.float64, False), (2, np.float32, True),
                                             (3, np.float64, True)])
def test_zslab_gloo_matches_single_domain(world, dtype, two):
    mp.spawn(_worker, args=(world, _free_port(), dtype, two, 3), nprocs=world, join=True)


def test_layout_bookkeeping():
    from paper_1606_02862_b200.pic.decomp import SlabLayout
    lay = SlabLayout(nx=16, ny=16, nz=64, scz=4, world=4, rank=0)
    lay.validate()
    assert (lay.nzl, lay.gp, lay.nze, lay.lower, lay.upper) == (16, 4, 24, 3, 1)
    assert lay.global_z(0) == 60 and lay.global_z(4) == 0 and lay.global_z(23) == 19
    assert lay.guard_layers() == ((0, 1), (5, 6))
    SlabLayout(16, 16, 64, 4, 8, 0).validate()          # 8-plane slabs, 4 guard planes
    with pytest.raises(ValueError):
        SlabLayout(16, 16, 12, 4, 2, 0).validate()      # 6-plane slab: not whole super cells
    SlabLayout(16, 16, 12, 4, 3, 0).validate()          # 4-plane slabs == guard depth: allowed
    with pytest.raises(ValueError):
        SlabLayout(16, 16, 8, 4, 4, 0).validate()       # 2-plane slabs: not whole super cells
    with pytest.raises(ValueError):
        SlabLayout(16, 16, 13, 4, 2, 0).validate()      # not divisible


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_j_plane_owners_cover_every_plane(world):
    """Fused J halo plane table (kwb_particles_advance_zslab): owned planes
    map to themselves, guard planes to the neighbour's owned plane of the same
    global z, and each global plane receives from exactly 1 + (guard copies)
    local planes -- the same sums _exchange_j performs."""
    from paper_1606_02862_b200.pic.decomp import SlabLayout, j_plane_owners
    nz, scz = 8 * world, 4
    lays = [SlabLayout(4, 4, nz, scz, world, r) for r in range(world)]
    hits = np.zeros(nz, dtype=int)
    for lay in lays:
        own = lay.owned()
        for zl, (o, oz) in enumerate(j_plane_owners(lay)):
            olay = lays[o]
            assert olay.owned().start <= oz < olay.owned().stop
            assert int(olay.global_z(oz)) == int(lay.global_z(zl))
            if own.start <= zl < own.stop:
                assert (o, oz) == (lay.rank, zl)
            hits[int(lay.global_z(zl))] += 1
    # every global plane: its owner plus the guard planes that cover it
    gp = lays[0].gp
    assert hits.sum() == world * (nz // world + 2 * gp)
    assert (hits >= 1).all()


def test_fuse_j_needs_cuda_slabs():
    """fuse_j=True is refused for slabs without device memory (the oracle
    locals): the plane table and peer mappings need CUDA buffers.  The
    default (None) falls back to the message exchange."""
    from oracle_slab import OracleLocal
    from paper_1606_02862_b200.pic import SimParams, default_species
    from paper_1606_02862_b200.pic.decomp import DecomposedSimulation, LoopbackTransport
    p = SimParams(cells=(8, 8, 16), species=default_species(2, 4.0), particles_per_cell=2,
                  dtype=np.dtype(np.float64))
    with pytest.raises(ValueError, match="fuse_j"):
        DecomposedSimulation(p, 2, range(2), LoopbackTransport(), local_factory=OracleLocal,
                             fuse_j=True)
    dec = DecomposedSimulation(p, 2, range(2), LoopbackTransport(), local_factory=OracleLocal)
    assert dec.fuse_j is False
