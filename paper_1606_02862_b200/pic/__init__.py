"""Drop-in for kernelweave.pic: SimParams, Species, Simulation, init_khi, ..."""

from .fields import (ALL_COMPONENTS, STAGGER, YeeFieldSet, div_b, div_j, field_energy,
                     tsc_weights, yee_dispersion_omega)
from .params import CFL_FACTOR, SHAPES, SimParams, Species, cfl_limit, default_dt, default_species
from .particles import SuperCellStore
from .pusher import MacroParticle, boris_push, lorentz_gamma, move_particle
from .sim import STRATEGIES, Simulation, diagnostics, init_khi, step

__all__ = [
    "ALL_COMPONENTS", "STAGGER", "YeeFieldSet", "div_b", "div_j", "field_energy",
    "tsc_weights", "yee_dispersion_omega", "CFL_FACTOR", "SHAPES", "SimParams", "Species",
    "cfl_limit", "default_dt", "default_species", "SuperCellStore", "MacroParticle",
    "boris_push", "lorentz_gamma", "move_particle", "STRATEGIES", "Simulation",
    "diagnostics", "init_khi", "step",
]
