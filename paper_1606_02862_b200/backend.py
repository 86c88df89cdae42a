"""The single execution back-end of this build: one B200 (sm_100a).

Stands where the reference's Backend plugins stand (kw/backends.py:68-308,
``make_backend``), but there is exactly one kind and no CPU fallback: a
Simulation given any other back-end raises CapabilityError."""

from __future__ import annotations

import torch

from .errors import CapabilityError


class B200Backend:
    kind = "b200"

    def __init__(self, device=None):
        if not torch.cuda.is_available():
            raise CapabilityError("B200Backend needs a CUDA device (none visible)")
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise CapabilityError(f"B200Backend needs a CUDA device, got {self.device}")
        major, minor = torch.cuda.get_device_capability(self.device)
        if (major, minor) != (10, 0):
            raise CapabilityError(
                f"libkwb200 is built for sm_100a (B200); device {self.device} is sm_{major}{minor}")
        self.worker_count = torch.cuda.get_device_properties(self.device).multi_processor_count

    def __repr__(self):
        return f"B200Backend({self.device})"


_BACKENDS = {"b200": B200Backend}


def make_backend(name: str = "b200", **kw):
    try:
        return _BACKENDS[name](**kw)
    except KeyError:
        raise CapabilityError(f"unknown backend {name!r}; this build provides only 'b200'") from None
