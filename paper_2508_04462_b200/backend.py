"""Operator plug-in (mirrors backend.py:20-66 of the reference).

The reference selects between a Cython module and a pure-Python mirror;
here there is exactly one backend, ``"b200"``, whose two protocol
functions launch CUDA kernels (csrc/card_ops.cu).  Selecting anything
else is a ConfigError — there is deliberately no CPU fallback.
"""

from __future__ import annotations

import types

import numpy as np
import torch

from ._device import ptr, require_cuda, stream_ptr, to_device
from ._lib import lib
from .errors import ConfigError, InputError, raise_for_status

BACKEND_NAME = "b200"


def kgram_dist(seed: int, seed2: int, mix_weight: float, tail, vocab_size: int, sharpness: float,
               temperature: float) -> np.ndarray:
    """_kernels.pyx:44-93 on the device: one (V,) float64 distribution."""
    out = kgram_dist_rows(seed, seed2, mix_weight, [tuple(tail)], vocab_size, sharpness, temperature)
    return out[0].cpu().numpy()


def kgram_dist_rows(seed, seed2, mix_weight, tails, vocab_size, sharpness, temperature,
                    out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched device form: tails is [n_rows][order] (equal lengths)."""
    dev = require_cuda()
    n = len(tails)
    L = len(tails[0]) if n else 0
    t = to_device(np.asarray(tails, dtype=np.int32).reshape(n, L), np.int32)
    if out is None:
        out = torch.empty((n, vocab_size), dtype=torch.float64, device=dev)
    M64 = (1 << 64) - 1
    rc = lib().card_kgram_dist(int(seed) & M64, int(seed2) & M64, float(mix_weight), ptr(t), L, L, n,
                               int(vocab_size), float(sharpness), float(temperature), ptr(out), stream_ptr())
    raise_for_status(rc, "card_kgram_dist")
    return out


def rows_topk(dists, k: int) -> list[list[tuple[int, float]]]:
    """_kernels.pyx:96-145 on the device."""
    d = np.asarray(dists, dtype=np.float64)
    if d.ndim != 2:
        raise InputError(f"rows_topk expects a 2-D array, got shape {d.shape}")
    n, V = d.shape
    if n == 0:
        return []
    kk = min(int(k), V)
    if kk <= 0:
        return [[] for _ in range(n)]
    dev = to_device(d, np.float64)
    tok = torch.empty((n, kk), dtype=torch.int32, device=dev.device)
    p = torch.empty((n, kk), dtype=torch.float64, device=dev.device)
    cnt = torch.empty(n, dtype=torch.int32, device=dev.device)
    rc = lib().card_rows_topk(ptr(dev), n, V, kk, ptr(tok), ptr(p), ptr(cnt), None, stream_ptr())
    raise_for_status(rc, "card_rows_topk")
    tok, p, cnt = tok.cpu().tolist(), p.cpu().tolist(), cnt.cpu().tolist()
    return [[(tok[i][j], p[i][j]) for j in range(cnt[i])] for i in range(n)]


_module = types.SimpleNamespace(BACKEND_NAME=BACKEND_NAME, kgram_dist=kgram_dist, rows_topk=rows_topk,
                                kgram_dist_rows=kgram_dist_rows)


def get_kernels():
    """Return the active kernel module (backend.py:42-47)."""
    return _module


def set_backend(name: str):
    if name != BACKEND_NAME:
        raise ConfigError(f"unknown kernel backend {name!r} (only {BACKEND_NAME!r} exists; no CPU fallback)")
    return _module


def active_backend_name() -> str:
    return BACKEND_NAME


def compiled_available() -> bool:
    try:
        lib()
    except Exception:
        return False
    return True
