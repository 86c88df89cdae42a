"""The split advance (kwb_particles_advance_split: a dense gather/push/move
kernel, then the deposit/shift kernel; csrc/push.cuh) against the oracle and
against the fused advance.

Bars: particles bitwise vs the oracle (as test_gpu_parity.py); fields within
the same stated bars; split vs fused on the GPU bitwise in particles.
"""

import numpy as np
import pytest

from golden_util import CASES, load_case
from parity_util import (FIELDS9, TOL_1STEP, assert_particles_bitwise, check_fields, make_pair,
                         order_spread)

pytestmark = pytest.mark.gpu


def _dtype(meta):
    return np.dtype(meta["config"]["dtype"])


@pytest.mark.parametrize("shape", ["tsc", "cic"])
@pytest.mark.parametrize("name", CASES)
def test_split_teacher_forced_vs_oracle(name, shape, monkeypatch):
    monkeypatch.setenv("KWB_SPLIT", "1")
    meta, _ = load_case(name)
    gpu, orc = make_pair(meta, shape=shape, validate=False)
    assert gpu.split_advance
    orc.run(2)
    gpu.load_state(fields={n: getattr(orc.fields, n) for n in FIELDS9},
                   particles=[st.packed() for st in orc.stores])
    spread = order_spread(orc)
    gpu.step()
    orc.step()
    for gs, os_ in zip(gpu.stores, orc.stores):
        assert_particles_bitwise(gs, os_)
    check_fields(f"{name}:split:{shape}", gpu.fields, lambda n: getattr(orc.fields, n),
                 TOL_1STEP[_dtype(meta)], spread=spread)


@pytest.mark.parametrize("name", ["khi_pair_f32", "thermal_e_f64", "eion_f32", "c2p_f32"])
def test_split_equals_fused(name, monkeypatch):
    """One step each way from the same state: identical stores, and fields
    within the stated bars of each other (J's shared-memory atomics make its
    summation order run-dependent in either path)."""
    meta, _ = load_case(name)
    sims = []
    for split in ("0", "1"):
        monkeypatch.setenv("KWB_SPLIT", split)
        gpu, orc = make_pair(meta, validate=True)
        assert gpu.split_advance == (split == "1")
        spread = order_spread(orc)
        gpu.step()
        sims.append(gpu)
    a, b = sims
    for sa, sb in zip(a.stores, b.stores):
        assert_particles_bitwise(sa, sb)
    check_fields(f"{name}:split_vs_fused", b.fields, lambda n: a.fields.numpy(n),
                 TOL_1STEP[_dtype(meta)], spread=spread)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_split_contract_violation(dtype, monkeypatch):
    """A particle moving a full cell raises before the field update."""
    monkeypatch.setenv("KWB_SPLIT", "1")
    from paper_1606_02862_b200.errors import ContractViolation
    from paper_1606_02862_b200.pic import SimParams, Simulation, Species
    p = SimParams(cells=(16, 16, 8), species=(Species("e", -1.0, 1.0, 1.0),), dtype=dtype)
    sim = Simulation(p, validate=False)
    assert sim.split_advance
    a = lambda *v: np.array(v, dtype=dtype)
    pk = dict(cx=np.array([3, 5]), cy=np.array([3, 5]), cz=np.array([1, 2]),
              ox=a(0.5, 3.0), oy=a(0.5, 0.5), oz=a(0.5, 0.5),
              ux=a(0, 0), uy=a(0, 0), uz=a(0, 0), w=a(1, 1))
    sim.load_state(particles=[pk])
    with pytest.raises(ContractViolation, match="1 particle"):
        sim.step()


@pytest.mark.parametrize("fuse_j", [False, True])
def test_split_in_zslab_decomposition(fuse_j, monkeypatch):
    """The split advance under the z-slab decomposition (two loopback slabs,
    message or fused J halo) against the single domain, as
    test_gpu_decomp.py checks the fused advance."""
    monkeypatch.setenv("KWB_SPLIT", "1")
    from test_gpu_decomp import test_loopback_slabs_match_single_domain
    test_loopback_slabs_match_single_domain(2, np.float32, "tsc", fuse_j)
