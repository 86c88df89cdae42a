"""paper_1606_02862_b200: a B200-native PIC cycle behind the kernelweave.pic API.

The hot path -- trilinear gather, relativistic Boris push, move, Esirkepov
deposit (CIC/TSC/PCS), super-cell shift and Yee field update -- runs as
hand-written sm_100a CUDA kernels in libkwb200.so (C ABI: include/kwb200.h),
called from the Python API in ``paper_1606_02862_b200.pic`` with PyTorch
owning the device memory.
"""

from .backend import B200Backend, make_backend
from .errors import (AllocationError, BufferMismatchError, CapabilityError,
                     ContractViolation, KernelWeaveError, NativeLibraryError)
from .workdiv import Extent3, WorkDivision, delinearize_3d, linearize_3d, make_work_division

__version__ = "0.1.0"

__all__ = [
    "B200Backend", "make_backend", "AllocationError", "BufferMismatchError",
    "CapabilityError", "ContractViolation", "KernelWeaveError", "NativeLibraryError",
    "Extent3", "WorkDivision", "delinearize_3d", "linearize_3d", "make_work_division",
]
