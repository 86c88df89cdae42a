"""khi-bench CLI: flags, presets, flop model, report
emission (CPU); one small validated run on the GPU."""

import csv
import io
import json

import pytest

from paper_1606_02862_b200 import cli


def test_presets_and_flop_model():
    assert cli.device_preset("k80") == (4350.0, 1450.0)
    assert cli.device_preset("Haswell") == (2354.0, 1177.0)
    with pytest.raises(ValueError, match="presets"):
        cli.device_preset("nope")
    assert cli.estimate_flops(0, 10, 10) == 0
    assert cli.estimate_flops(2, 100, 10) == 2 * cli.estimate_flops(1, 100, 10)


def test_report_emission_roundtrip():
    rec = {k: 0 for k in cli.FIELDS}
    rec.update(backend="b200", strategy="elements", precision="f64")
    text = cli.emit_report([rec], "csv")
    rows = list(csv.DictReader(io.StringIO(text)))
    assert list(rows[0].keys()) == list(cli.FIELDS)
    assert cli.emit_report([rec], "csv") == text                # byte-identical re-emission
    assert json.loads(cli.emit_report([rec], "json"))["records"][0]["backend"] == "b200"
    assert cli.emit_report([], "csv") == ",".join(cli.FIELDS) + "\n"


def test_cpu_backends_rejected():
    with pytest.raises(SystemExit):
        cli.parse_args(["--backend", "serial"])
    with pytest.raises(SystemExit):
        cli.parse_args(["--reps", "0"])


@pytest.mark.gpu
def test_cli_small_run(tmp_path):
    out = tmp_path / "r.json"
    ck = tmp_path / "end.kwpic"
    rc = cli.main(["--cells", "16", "--steps", "5", "--ppc", "4", "--precision", "f64",
                   "--thermal-u", "0.05", "--format", "json", "--out", str(out),
                   "--checkpoint", str(ck)])
    assert rc == 0
    rec = json.loads(out.read_text())["records"][0]
    assert rec["particles"] == 16 ** 3 * 4 * 2
    assert rec["max_continuity_residual"] <= 1e-12
    assert ck.exists()
