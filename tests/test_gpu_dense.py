"""Dense and hot plasma against the oracle: 40 particles per cell per species
and thermal_u 0.3 (about a third of the particles cross a cell face per
step), so every warp queue of the advance kernel fills several times within
one launch -- the mid-loop drains of the CIC/TSC crossing queue and the
wrap-around of the PCS ring (64 records, drained 32 at a time) -- at the
float32 PCS instance's 3 CTAs per SM.  One teacher-forced step: particles
bitwise, J within the float32 one-step bar, charge conserved."""

from __future__ import annotations

import numpy as np
import pytest

from golden_util import rel_l2
from parity_util import TOL_1STEP, TOL_RESID, assert_particles_bitwise, check_fields, order_spread

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", ["cic", "tsc", "pcs"])
def test_dense_hot_plasma_one_step(shape):
    from oracle.pic import oracle_init_khi
    from paper_1606_02862_b200.pic import SimParams, default_species, init_khi

    order = {"cic": 1, "tsc": 2, "pcs": 3}[shape]
    p = SimParams(cells=(16, 16, 8), species=default_species(40, 1836.0),
                  particles_per_cell=40, dtype=np.float32, stream_velocity=0.0,
                  perturbation=0.0, thermal_u=0.3, shape=shape)
    gpu = init_khi(p, seed=21, validate=True)
    orc = oracle_init_khi(p, seed=21, validate=True, shape_order=order, threads=8)
    for it in range(2):
        if it:
            gpu.load_state(fields={n: getattr(orc.fields, n) for n in
                                   ("Ex", "Ey", "Ez", "Bx", "By", "Bz", "Jx", "Jy", "Jz")},
                           particles=[st.packed() for st in orc.stores])
        spread = order_spread(orc)
        gpu.step()
        orc.step()
        for gs, os_ in zip(gpu.stores, orc.stores):
            assert_particles_bitwise(gs, os_)
        check_fields(f"dense_{shape}:step{it}", gpu.fields, lambda n: getattr(orc.fields, n),
                     TOL_1STEP[np.dtype(np.float32)], names=("Jx", "Jy", "Jz"), spread=spread)
        assert gpu.last_residual <= TOL_RESID[np.dtype(np.float32)]
