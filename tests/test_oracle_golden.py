"""Pin the CPU oracle to the unmodified reference (golden dumps).

The oracle (oracle/pic.py + pic_oracle.c) must reproduce kernelweave.pic's
Serial back-end BITWISE: particle records in canonical order, all nine field
lattices, the validation charge density and the continuity residual, over
several free-running steps, for fp64 and fp32, one and two species,
anisotropic cells and a non-default super cell.
"""

import json
import os

import numpy as np
import pytest

from golden_util import CASES, GOLDEN, digest, load_case, oracle_params

FIELDS9 = ("Ex", "Ey", "Ez", "Bx", "By", "Bz", "Jx", "Jy", "Jz")


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_bitwise(name, oracle_lib):
    meta, data = load_case(name)
    p = oracle_params(meta)
    sim = oracle_lib.oracle_init_khi(p, seed=meta["config"]["seed"], validate=True, threads=4)
    steps = sorted(int(k[1:]) for k in meta["steps"])
    for t in range(max(steps) + 1):
        if t in steps:
            key = f"t{t}"
            sm = meta["steps"][key]
            assert sim.census() == sm["census"]
            for i, st in enumerate(sim.stores):
                pk = st.packed()
                for k, v in pk.items():
                    assert digest(v) == sm["species"][i][k], (key, i, k)
                np.testing.assert_array_equal(st.super_cell_counts(), data[f"{key}_s{i}_sc_counts"])
            for n in FIELDS9:
                np.testing.assert_array_equal(getattr(sim.fields, n), data[f"{key}_{n}"], err_msg=n)
            np.testing.assert_array_equal(sim.charge_density(), data[f"{key}_rho"])
            if t > 0:
                assert sim.last_residual == sm["residual"]
                d = sim.diagnostics()
                for k2, v2 in sm["diagnostics"].items():
                    assert d[k2] == pytest.approx(v2, rel=1e-12, abs=1e-300), k2
        if t < max(steps):
            sim.step()


def test_oracle_thread_count_invariant(oracle_lib):
    """Tiles are computed in parallel but merged in super-cell order, so the
    oracle is bitwise independent of its thread count."""
    meta, _ = load_case("khi_pair_f32")
    p = oracle_params(meta)
    a = oracle_lib.oracle_init_khi(p, seed=3, threads=1)
    b = oracle_lib.oracle_init_khi(p, seed=3, threads=8)
    a.run(2)
    b.run(2)
    for n in FIELDS9:
        np.testing.assert_array_equal(getattr(a.fields, n), getattr(b.fields, n))
    for sa, sb in zip(a.stores, b.stores):
        for k, v in sa.packed().items():
            np.testing.assert_array_equal(v, sb.packed()[k])


def test_kat_shapes_and_boris(oracle_lib):
    """SPEC.md known answers, computed by the reference into kat.json."""
    with open(os.path.join(GOLDEN, "kat.json")) as fh:
        kat = json.load(fh)
    assert kat["tsc_half"] == [0.125, 0.75, 0.125]
    assert sum(kat["tsc_half"]) == 1.0
    # Boris with B = 0: u' = u + q dt E / m exactly
    u, e, q, m, dt = (0.1, -0.2, 0.3), (0.5, 0.0, 0.0), -1.0, 1.0, 0.5
    qm = q * dt / (2.0 * m)
    assert kat["boris_b0"][1] == u[1] and kat["boris_b0"][2] == u[2]
    assert kat["boris_b0"][0] == pytest.approx(u[0] + 2 * qm * e[0], abs=1e-16)


def test_shared_reciprocal_division_is_ieee_division():
    """The CUDA push/move divide three numerators by one divisor through
    r = 1/b and a Markstein correction (csrc/advance.cuh div_rcp); bit for
    bit IEEE a / b over 2^24 pairs drawn like the kernel's operands (C99
    fma, the same IEEE operation as __fma_rn)."""
    from oracle import pic as orc
    assert orc.lib().orc_div_rcp_check(1 << 24, 12345) == 0
    # the PCS weights' a / 6 through the same construction (csrc/advance.cuh div6)
    assert orc.lib().orc_div6_check(1 << 24, 777) == 0


@pytest.mark.parametrize("name", ["c1_tsc_f64", "c1_tsc_f32", "c2p_f32", "c3p_f32", "c4p_f32"])
def test_oracle_matches_reference_at_baseline_scale(name, oracle_lib):
    """BASELINE scale: C1 in full (32^3 x 8 ppc, 100 steps) in fp64 and fp32
    and 32^3 proxies of C2 (25 ppc e/ion 1836), C3 (16 ppc KHI pair) and C4
    (32 ppc electrons), 10 steps.  The oracle reproduces the reference's
    digests of every lattice and every packed particle array at each dumped
    step bit for bit, plus occupancy, super-cell counts, the continuity
    residual and diagnostics -- so the GPU tests may compare against the
    oracle at these sizes (tests/test_gpu_scale.py)."""
    meta, data = load_case(name)
    p = oracle_params(meta)
    sim = oracle_lib.oracle_init_khi(p, seed=meta["config"]["seed"], validate=True)
    steps = sorted(int(k[1:]) for k in meta["steps"])
    for t in range(max(steps) + 1):
        if t in steps:
            key = f"t{t}"
            sm = meta["steps"][key]
            assert sim.census() == sm["census"]
            for i, st in enumerate(sim.stores):
                pk = st.packed()
                for k, v in pk.items():
                    assert digest(v) == sm["species"][i][k], (key, i, k)
                np.testing.assert_array_equal(st.super_cell_counts(), data[f"{key}_s{i}_sc_counts"])
            for n in FIELDS9:
                assert digest(getattr(sim.fields, n)) == sm["fields"][n], (key, n)
            if t > 0:
                assert sim.last_residual == sm["residual"]
        if t < max(steps):
            sim.step()
