"""khi-bench: the benchmark/validation CLI the reference declares but does
not ship (pkg/pyproject.toml:18-19 -> kernelweave.cli:main, missing; spec in
SPEC.md:549-606).  Runs the KHI simulation on the B200 and reports runtime,
particle-updates/s and an analytic floating-point efficiency as CSV or JSON.

    python -m paper_1606_02862_b200.cli --cells 32 --steps 100 --ppc 16 \\
        --precision f64 --format json --out report.json --checkpoint end.kwpic

Flags follow SPEC.md:601.  ``--backend`` accepts only ``b200`` (the
reference's serial/blockpool/coop CPU back-ends are not part of this build
and are rejected with a message); ``--workers`` and ``--strategy`` are
accepted for command-line compatibility.  Exit code is non-zero if any run
fails validation (continuity residual above 1e-12 in f64 / 1e-6 in f32).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import sys
import time

import numpy as np

# PAPER.md Table 1 peak GFLOPS (sp, dp); "b200" = measured on this pool's
# B200s (profiles/r01_microbench.txt: FFMA 3.26e13 FMA/s, DMUL/DADD 1.83e13/s).
PRESETS = {
    "k80": (4350.0, 1450.0),
    "haswell": (2354.0, 1177.0),
    "power8": (1120.0, 560.0),
    "interlagos": (960.0, 480.0),
    "b200": (65200.0, 36600.0),
}

# Analytic flop counts per particle and per cell per PIC cycle, counted from
# the arithmetic of the reference kernels (pic/kernels.py) for a particle that
# does not cross a cell face: gather 6 x 21 + 6, Boris push 61 (each divide
# and sqrt counted as one flop), move 25, TSC Esirkepov deposit 202;
# Faraday 2 x 21 and Ampere 24 per cell.
C_PARTICLE = 132 + 61 + 25 + 202
C_FIELD = 2 * 21 + 24

FIELDS = ("backend", "strategy", "precision", "cells", "particles", "steps", "wall_seconds",
          "particle_updates_per_second", "estimated_flops", "achieved_gflops",
          "efficiency_percent", "max_continuity_residual", "energy_drift_percent")


def estimate_flops(steps: int, particles: int, cells: int) -> int:
    """steps * (particles * C_PARTICLE + cells * C_FIELD)."""
    return int(steps) * (int(particles) * C_PARTICLE + int(cells) * C_FIELD)


def device_preset(name: str):
    try:
        return PRESETS[name.lower()]
    except KeyError:
        raise ValueError(f"unknown preset {name!r}; presets: {', '.join(PRESETS)}") from None


def run_benchmark(cfg) -> dict:
    from .pic import SimParams, default_species, init_khi
    dtype = np.float32 if cfg.precision == "f32" else np.float64
    p = SimParams(cells=(cfg.cells,) * 3, species=default_species(cfg.ppc, cfg.mass_ratio),
                  particles_per_cell=cfg.ppc, dtype=dtype, shape=cfg.shape,
                  thermal_u=cfg.thermal_u)
    sim = init_khi(p, seed=cfg.seed, strategy=cfg.strategy, validate=not cfg.no_validate)
    e0 = sim.total_energy()
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    max_res = 0.0
    for _ in range(cfg.steps):
        sim.step()
        if sim.validate:
            max_res = max(max_res, sim.last_residual)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    e1 = sim.total_energy()
    n_p = sim.census()
    flops = estimate_flops(cfg.steps, n_p, p.cells.volume)
    peak = cfg.peak_sp if cfg.precision == "f32" else cfg.peak_dp
    gflops = flops / wall / 1e9 if wall > 0 else 0.0
    rec = {
        "backend": cfg.backend, "strategy": cfg.strategy, "precision": cfg.precision,
        "cells": cfg.cells, "particles": n_p, "steps": cfg.steps, "wall_seconds": wall,
        "particle_updates_per_second": n_p * cfg.steps / wall if wall > 0 else 0.0,
        "estimated_flops": flops, "achieved_gflops": gflops,
        "efficiency_percent": 100.0 * gflops / peak if peak else 0.0,
        "max_continuity_residual": max_res,
        "energy_drift_percent": 100.0 * (e1 - e0) / e0 if e0 else 0.0,
    }
    if cfg.checkpoint:
        from .pic.checkpoint import save_checkpoint
        save_checkpoint(sim, cfg.checkpoint)
    return rec


def emit_report(records, fmt: str) -> str:
    if fmt == "json":
        return json.dumps({"records": records, "flop_model": {
            "C_particle": C_PARTICLE, "C_field": C_FIELD,
            "method": "analytic count of the reference kernels' arithmetic"}}, indent=1) + "\n"
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=FIELDS, lineterminator="\n")
    w.writeheader()
    for r in records:
        w.writerow(r)
    return buf.getvalue()


def parse_args(argv=None):
    ap = argparse.ArgumentParser(prog="khi-bench", description=__doc__.split("\n\n")[0])
    ap.add_argument("--backend", default="b200")
    ap.add_argument("--workers", type=int, default=int(os.environ.get("KW_WORKERS", "0") or 0))
    ap.add_argument("--strategy", default="elements", choices=("elements", "threads"))
    ap.add_argument("--cells", type=int, default=32)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--ppc", type=int, default=16)
    ap.add_argument("--precision", default="f64", choices=("f32", "f64"))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--preset", default=None)
    ap.add_argument("--peak-sp", type=float, default=None)
    ap.add_argument("--peak-dp", type=float, default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--format", default="csv", choices=("csv", "json"))
    ap.add_argument("--checkpoint", default=None)
    ap.add_argument("--shape", default="tsc", choices=("cic", "tsc", "pcs"))
    ap.add_argument("--mass-ratio", type=float, default=1.0)
    ap.add_argument("--thermal-u", type=float, default=0.0)
    ap.add_argument("--no-validate", action="store_true")
    cfg = ap.parse_args(argv)
    if cfg.reps < 1:
        ap.error("--reps must be >= 1")
    if cfg.backend != "b200":
        ap.error(f"backend {cfg.backend!r} is a CPU back-end of the reference; "
                 "this build runs on 'b200' only")
    sp, dp = device_preset(cfg.preset or "b200")
    cfg.peak_sp = cfg.peak_sp or sp
    cfg.peak_dp = cfg.peak_dp or dp
    if cfg.peak_sp <= 0 or cfg.peak_dp <= 0:
        ap.error("peak GFLOPS must be > 0")
    return cfg


def main(argv=None) -> int:
    cfg = parse_args(argv)
    runs = [run_benchmark(cfg) for _ in range(cfg.reps)]
    runs.sort(key=lambda r: r["wall_seconds"])
    rec = runs[len(runs) // 2]  # median repetition
    text = emit_report([rec], cfg.format)
    if cfg.out:
        with open(cfg.out, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    limit = 1e-6 if cfg.precision == "f32" else 1e-12
    ok = cfg.no_validate or rec["max_continuity_residual"] <= limit
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
