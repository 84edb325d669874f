"""Chain verification API (mirrors verify.py:27-132 of the reference).

Each call runs the device accept-and-correct kernel (csrc/card_engine.cu:
verify_probs_kernel) on uploaded fp64 distributions.  Randomness stays the
caller's numpy Generator: the kernel is fed uniforms drawn from a copy of
its state and the generator is then advanced by exactly the number the
kernel consumed, so the stream matches sequential ``rng.random()`` calls.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from ._device import ptr, require_cuda, stream_ptr, to_device
from ._lib import EngineState, lib
from .errors import InputError, ProtocolError, raise_for_status

TokenId = int


@dataclass(frozen=True)
class VerifyOutcome:
    accepted: tuple
    correction: TokenId
    accepted_len: int
    lnew: int

    @property
    def committed(self) -> tuple:
        return self.accepted + (self.correction,)


def _check_inputs(target_dists, candidate) -> None:
    if len(target_dists) != len(candidate) + 1:
        raise InputError(f"need len(candidate)+1 target distributions, got {len(target_dists)} "
                         f"for {len(candidate)} candidate tokens")
    for i, tok in enumerate(candidate):
        if not isinstance(tok, (int, np.integer)) or tok < 0 or tok >= len(target_dists[i]):
            raise InputError(f"candidate token {tok!r} at position {i} is out of vocabulary")


def _run(dists, candidate, sampling: bool, q=None, uniforms=None):
    dev = require_cuda()
    d = np.ascontiguousarray(np.vstack([np.asarray(x, dtype=np.float64) for x in dists]))
    L = len(candidate)
    st = EngineState()
    st.L = L
    st.sampling = int(sampling)
    st.hit = 1 if L else 0
    E = torch.frombuffer(bytearray(bytes(st)), dtype=torch.int32).to(dev)
    cand = to_device(np.asarray(list(candidate) + [0], dtype=np.int32), np.int32)
    dd = to_device(d, np.float64)
    qd = to_device(np.asarray(q, dtype=np.float64), np.float64) if q is not None and L else None
    uni = to_device(np.asarray(uniforms if uniforms is not None else [0.0], dtype=np.float64), np.float64)
    rc = lib().card_verify_probs(ptr(E), ptr(cand), ptr(dd), d.shape[1], ptr(qd), ptr(uni), stream_ptr())
    raise_for_status(rc, "card_verify_probs")
    out = EngineState.from_buffer_copy(E.cpu().numpy().tobytes())
    n = out.n_acc
    return tuple(int(t) for t in candidate[:n]), int(out.corr), out.cursor


def argmax_token(probs) -> TokenId:
    """First maximum (verify.py:38-40), on the device."""
    _, corr, _ = _run([probs], [], False)
    return corr


def sample_index(rng: np.random.Generator, probs) -> TokenId:
    """CDF inversion with one uniform (verify.py:43-51), on the device."""
    p = np.asarray(probs, dtype=np.float64)
    total = float(np.cumsum(p)[-1]) if p.size else 0.0
    if not np.isfinite(total) or total <= 0.0:
        raise InputError("cannot sample from an all-zero distribution")
    u = rng.random()
    _, corr, _ = _run([p], [], True, uniforms=[u])
    return corr


def verify_greedy(target_dists: Sequence, candidate: Sequence[TokenId]) -> VerifyOutcome:
    """Longest argmax prefix + correction (verify.py:65-80)."""
    _check_inputs(target_dists, candidate)
    acc, corr, _ = _run(target_dists, list(candidate), False)
    return VerifyOutcome(accepted=acc, correction=corr, accepted_len=len(acc), lnew=len(acc) + 1)


def verify_sampling(target_dists: Sequence, draft_conditionals: Sequence[float], candidate: Sequence[TokenId],
                    rng: np.random.Generator) -> VerifyOutcome:
    """Lossless accept/reject (verify.py:83-132)."""
    _check_inputs(target_dists, candidate)
    if len(draft_conditionals) != len(candidate):
        raise InputError(f"need one draft conditional per candidate token, got {len(draft_conditionals)} "
                         f"for {len(candidate)}")
    # the reference checks a conditional only when the walk reaches its
    # position (verify.py:104-112): verify up to the first invalid one and
    # raise only if every position before it was accepted
    bad = next((i for i, q in enumerate(draft_conditionals) if not np.isfinite(float(q)) or float(q) <= 0.0),
               None)
    cand = list(candidate) if bad is None else list(candidate[:bad])
    dists = list(target_dists) if bad is None else list(target_dists[:bad + 1])
    qs = [float(q) for q in draft_conditionals[:len(cand)]]
    saved = rng.bit_generator.state
    uni = rng.random(len(cand) + 2)
    acc, corr, used = _run(dists, cand, True, q=qs, uniforms=uni)
    rng.bit_generator.state = saved
    if bad is not None and len(acc) == bad:
        if bad:
            rng.random(bad)   # the coins of the accepted positions were drawn before the check
        q = float(draft_conditionals[bad])
        raise ProtocolError(f"draft conditional {q!r} at position {bad}: the cache proposed a token it "
                            f"assigned no probability")
    if used:
        rng.random(used)   # advance by exactly what the kernel consumed
    return VerifyOutcome(accepted=acc, correction=corr, accepted_len=len(acc), lnew=len(acc) + 1)
