"""Device plumbing: torch provides memory and streams; kernels live in
libcard_b200.so.  No CPU fallback — no GPU means DeviceError."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from .errors import DeviceError


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("a CUDA device (B200, sm_100a) is required; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream: torch.cuda.Stream | None = None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def to_device(a, dtype) -> torch.Tensor:
    dev = require_cuda()
    arr = np.ascontiguousarray(a, dtype=dtype)
    return torch.from_numpy(arr).to(dev, non_blocking=False)
