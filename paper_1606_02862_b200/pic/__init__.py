"""Drop-in for kernelweave.pic: SimParams, Species, Simulation, init_khi, ..."""

from .fields import (ALL_COMPONENTS, STAGGER, YeeFieldSet, div_b, div_j, field_energy,
                     gather_fields, tsc_weights, yee_dispersion_omega, yee_update_b,
                     yee_update_e)
from .params import CFL_FACTOR, SHAPES, SimParams, Species, cfl_limit, default_dt, default_species
from .particles import SuperCellStore
from .pusher import MacroParticle
from .sim import STRATEGIES, Simulation, diagnostics, init_khi, step

__all__ = [
    "ALL_COMPONENTS", "STAGGER", "YeeFieldSet", "div_b", "div_j", "field_energy",
    "gather_fields", "tsc_weights", "yee_dispersion_omega", "yee_update_b", "yee_update_e", "CFL_FACTOR", "SHAPES", "SimParams", "Species",
    "cfl_limit", "default_dt", "default_species", "SuperCellStore", "MacroParticle",
    "STRATEGIES", "Simulation",
    "diagnostics", "init_khi", "step",
]
