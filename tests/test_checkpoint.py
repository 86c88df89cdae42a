"""KWPIC1 checkpoint: format round trip on CPU, and on the GPU
byte-identical files for the GPU and oracle initial states plus a bitwise
restart (save -> load -> step == step)."""

import os

import numpy as np
import pytest

from paper_1606_02862_b200.pic.checkpoint import read_checkpoint, save_checkpoint

FIELDS9 = ("Ex", "Ey", "Ez", "Bx", "By", "Bz", "Jx", "Jy", "Jz")


def _params():
    from paper_1606_02862_b200.pic import SimParams, default_species
    return SimParams(cells=(16, 16, 8), species=default_species(4, 1836.0), particles_per_cell=4,
                     dtype=np.float32, stream_velocity=0.1, perturbation=0.02, thermal_u=0.1)


def test_oracle_checkpoint_roundtrip(tmp_path):
    from oracle.pic import oracle_init_khi
    p = _params()
    orc = oracle_init_khi(p, seed=4, validate=False, threads=2)
    orc.run(2)
    path = os.path.join(tmp_path, "o.kwpic")
    save_checkpoint(orc, path)
    c = read_checkpoint(path)
    assert c["cells"] == (16, 16, 8) and c["step_count"] == 2 and len(c["species"]) == 2
    for n in FIELDS9:
        np.testing.assert_array_equal(c["fields"][n], getattr(orc.fields, n))
    for i, st in enumerate(orc.stores):
        pk = st.packed()
        assert c["particles"][i]["cx"].shape == pk["cx"].shape
        assert int(c["particles"][i]["_counts"].sum()) == st.census()
        np.testing.assert_array_equal(np.sort(c["particles"][i]["ux"]), np.sort(pk["ux"]))
    # deterministic: writing the same state twice gives the same bytes
    path2 = os.path.join(tmp_path, "o2.kwpic")
    save_checkpoint(orc, path2)
    assert open(path, "rb").read() == open(path2, "rb").read()


@pytest.mark.gpu
def test_gpu_checkpoint_matches_oracle_and_restarts(tmp_path):
    from oracle.pic import oracle_init_khi
    from paper_1606_02862_b200.pic import init_khi
    from paper_1606_02862_b200.pic.checkpoint import load_checkpoint
    p = _params()
    gpu = init_khi(p, seed=4, validate=False)
    orc = oracle_init_khi(p, seed=4, validate=False, threads=2)
    a, b = os.path.join(tmp_path, "g.kwpic"), os.path.join(tmp_path, "o.kwpic")
    save_checkpoint(gpu, a)
    save_checkpoint(orc, b)
    assert open(a, "rb").read() == open(b, "rb").read()     # identical initial state
    gpu.step()
    save_checkpoint(gpu, a)
    restarted = load_checkpoint(a, validate=False)
    gpu.step()
    restarted.step()
    ca, cb = os.path.join(tmp_path, "a.kwpic"), os.path.join(tmp_path, "b.kwpic")
    save_checkpoint(gpu, ca)
    save_checkpoint(restarted, cb)
    x, y = read_checkpoint(ca), read_checkpoint(cb)
    for i in range(2):
        for k in ("cx", "cy", "cz", "ox", "ux", "w"):
            np.testing.assert_array_equal(x["particles"][i][k], y["particles"][i][k])
    for n in FIELDS9:
        d = np.linalg.norm(x["fields"][n] - y["fields"][n])
        assert d <= 1e-5 * max(np.linalg.norm(y["fields"][n]), 1e-30)
