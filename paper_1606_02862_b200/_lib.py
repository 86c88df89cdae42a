"""ctypes binding of libkwb200.so (the C ABI declared in include/kwb200.h).

There is no CPU fallback: if the library is missing or a call fails, a
NativeLibraryError is raised.  Structs mirror the header field for field.
"""

from __future__ import annotations

import ctypes
import os

from .errors import NativeLibraryError

_HERE = os.path.dirname(os.path.abspath(__file__))
# KWB_LIB_PATH overrides the library (A/B builds of the same ABI; never a CPU path)
LIB_PATH = os.environ.get("KWB_LIB_PATH") or os.path.join(_HERE, "libkwb200.so")

KWB_F32, KWB_F64 = 0, 1
ST_MOVE_ERRORS, ST_EXCH_OVERFLOW, ST_STORE_OVERFLOW, ST_LEAVERS, ST_MAX_COUNT, \
    ST_LOAD_ERRORS, ST_GUARD_OVERFLOW = range(7)
STATUS_WORDS = 8

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
D = ctypes.c_double


class Grid(ctypes.Structure):
    _fields_ = [("nx", I32), ("ny", I32), ("nz", I32),
                ("scx", I32), ("scy", I32), ("scz", I32),
                ("gx", I32), ("gy", I32), ("gz", I32),
                ("dtype", I32),
                ("dx", D), ("dy", D), ("dz", D), ("dt", D)]


class SpeciesC(ctypes.Structure):
    _fields_ = [("qm_half_dt", D), ("fac", D * 3), ("dt_d", D * 3),
                ("q_inv_vol", D), ("charge", D), ("mass", D)]


class StoreC(ctypes.Structure):
    _fields_ = [("ox", P), ("oy", P), ("oz", P), ("ux", P), ("uy", P), ("uz", P),
                ("w", P), ("front", P), ("back", P), ("frames_per_sc", I32)]


class ExchangeC(ctypes.Structure):
    _fields_ = [("ox", P), ("oy", P), ("oz", P), ("ux", P), ("uy", P), ("uz", P),
                ("w", P), ("cx", P), ("cy", P), ("cz", P), ("dest", P), ("count", P),
                ("capacity", I32)]


class InitC(ctypes.Structure):
    _fields_ = [("ppc", I32), ("px", I32), ("py", I32), ("pz", I32),
                ("stream_velocity", D), ("perturbation", D), ("thermal_u", D), ("weight", D),
                ("seed", ctypes.c_uint64), ("species_index", I32),
                ("x_offset", I32), ("y_offset", I32), ("z_offset", I32),
                ("global_nx", I32), ("global_ny", I32)]


Ptr3 = P * 3
Ptr7 = P * 7

_SIGS = {
    "kwb_version": ([], ctypes.c_int),
    "kwb_last_error": ([], ctypes.c_char_p),
    "kwb_particles_advance": ([P, P, P, P, P, Ptr3, Ptr3, Ptr3, ctypes.c_int, P, P],
                              ctypes.c_int),
    "kwb_particles_advance_zslab": ([P, P, P, P, P, Ptr3, Ptr3, Ptr3, P, ctypes.c_int, P, P],
                                    ctypes.c_int),
    "kwb_particles_shift": ([P, P, P, P, P], ctypes.c_int),
    "kwb_particles_advance_species": ([P, ctypes.c_int32, P, P, P, P, Ptr3, Ptr3, Ptr3, P,
                                       ctypes.c_int, P, P], ctypes.c_int),
    "kwb_particles_advance_split": ([P, ctypes.c_int32, P, P, P, P, P, Ptr3, Ptr3, Ptr3, P,
                                     ctypes.c_int, P, P], ctypes.c_int),
    "kwb_particles_shift_species": ([P, ctypes.c_int32, P, P, P, P], ctypes.c_int),
    "kwb_fields_faraday_half": ([P, Ptr3, Ptr3, D, P], ctypes.c_int),
    "kwb_fields_ampere": ([P, Ptr3, Ptr3, Ptr3, D, P], ctypes.c_int),
    "kwb_fields_gather": ([P, Ptr3, Ptr3, I64, P, P, P, P], ctypes.c_int),
    "kwb_zero_step": ([P, P, P, ctypes.c_int32, P], ctypes.c_int),
    "kwb_enable_peer_access": ([ctypes.c_int32], ctypes.c_int),
    "kwb_copy_async": ([P, P, I64, P], ctypes.c_int),
    "kwb_check_failures": ([ctypes.c_int32], ctypes.c_int64),
    "kwb_charge_density": ([P, P, P, ctypes.c_int, P, P], ctypes.c_int),
    "kwb_continuity_residual": ([P, P, P, Ptr3, Ptr3, P, P, P], ctypes.c_int),
    "kwb_particle_moments": ([P, P, P, P, P], ctypes.c_int),
    "kwb_field_stats": ([P, Ptr3, Ptr3, P, P], ctypes.c_int),
    "kwb_store_load": ([P, P, I64, P, P, P, Ptr7, P, P], ctypes.c_int),
    "kwb_store_export": ([P, P, I64, I64, P, ctypes.c_int, P, P, P, Ptr7, P], ctypes.c_int),
    "kwb_store_extract": ([P, P, I64, I64, P, I64, P, P, P, Ptr7, P, P, P], ctypes.c_int),
    "kwb_store_load_counted": ([P, P, P, I64, P, P, P, Ptr7, P, P], ctypes.c_int),
    "kwb_store_repack": ([P, P, P, P], ctypes.c_int),
    "kwb_init_khi": ([P, P, P, P], ctypes.c_int),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load libkwb200.so and declare every C-ABI signature."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.kwb_version() != 1:
        raise NativeLibraryError(f"libkwb200 ABI version {lib.kwb_version()} != 1")
    if path == LIB_PATH:
        _lib = lib
    return lib


def call(name: str, *args) -> None:
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.kwb_last_error().decode(errors="replace")
        raise NativeLibraryError(f"{name} failed ({rc}): {msg}")


def ptr(t) -> int:
    """Device pointer of a torch tensor (must be contiguous)."""
    return t.data_ptr()


def ptr3(ts) -> "Ptr3":
    return Ptr3(*(t.data_ptr() for t in ts))


def ptr7(ts) -> "Ptr7":
    return Ptr7(*(t.data_ptr() for t in ts))
