"""Query-and-correct decode loop on the device (mirrors engine.py:41-423 of
the reference).

Every protocol step is a CUDA kernel sequence on one stream:

  draft step  : card_draft_rows -> model forward (k-gram stream or
                transformer + lm_head top-k) -> card_cache_expand_topk ->
                card_record_width                       (engine.py:198-221)
  target step : card_cache_query -> card_target_rows -> model forward ->
                card_verify_{argmax,probs} -> card_commit -> card_cache_correct
                -> draft KV promote / compaction move -> card_cycle_end
                                                         (engine.py:228-272)

Two drivers share those sequences:

* ``stepwise`` (parity / trace mode): the host synchronises after every
  step, reproducing ``_run_serial`` (engine.py:290-317) event for event,
  including ``cache_alive_nodes`` and the virtual clock;
* ``graph`` (throughput mode): each step is a captured CUDA graph; the host
  launches ``min(ratio, max_depth - depth)`` draft graphs and one target
  graph per cycle and reads back one record per cycle (no other sync).

``mode="concurrent"`` runs the same lockstep schedule on one GPU: greedy
output is schedule-invariant (engine.py:11-12), the trace is the serial one.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import asdict, dataclass, field
from typing import Sequence

import numpy as np
import torch

from ._device import ptr, require_cuda, stream_ptr
from ._lib import EngineState, lib
from .cache import CacheConfig, TreeCache
from .errors import ConfigError, InputError, ProtocolError, raise_for_status
from .metrics import RunMetrics, finalize

TokenId = int
MODES = ("serial_sim", "concurrent")
PREFILL_CHUNK = 256


def communication_ratio(target_latency: float, draft_latency: float) -> int:
    """engine.py:41-48."""
    if target_latency <= 0.0 or draft_latency <= 0.0:
        raise ConfigError("latencies must be positive")
    return max(1, math.ceil(target_latency / draft_latency - 1e-9))


@dataclass
class EngineConfig:
    """engine.py:51-102 (same fields, defaults and validation)."""

    K: int = 50
    k: int = 3
    ratio: int = 5
    temperature: float = 0.0
    max_new_tokens: int = 64
    mode: str = "serial_sim"
    correction_enabled: bool = True
    seed: int = 0
    query_depth: int | None = None
    max_depth: int | None = None
    time_scale: float = 1e-3

    def __post_init__(self) -> None:
        for name in ("K", "k", "ratio", "max_new_tokens"):
            v = getattr(self, name)
            if not isinstance(v, int) or isinstance(v, bool) or v < 1:
                raise ConfigError(f"{name} must be a positive integer, got {v!r}")
        if self.query_depth is None:
            self.query_depth = self.ratio
        if self.max_depth is None:
            self.max_depth = 2 * self.ratio
        for name in ("query_depth", "max_depth"):
            v = getattr(self, name)
            if not isinstance(v, int) or isinstance(v, bool) or v < 1:
                raise ConfigError(f"{name} must be a positive integer, got {v!r}")
        if not isinstance(self.temperature, (int, float)) or not math.isfinite(self.temperature):
            raise ConfigError(f"temperature must be finite, got {self.temperature!r}")
        if self.temperature < 0.0:
            raise ConfigError(f"temperature must be >= 0, got {self.temperature!r}")
        if self.mode not in MODES:
            raise ConfigError(f"mode must be one of {MODES}, got {self.mode!r}")
        if not isinstance(self.seed, int) or isinstance(self.seed, bool):
            raise ConfigError(f"seed must be an integer, got {self.seed!r}")
        if not isinstance(self.time_scale, (int, float)) or self.time_scale <= 0.0:
            raise ConfigError(f"time_scale must be positive, got {self.time_scale!r}")
        if not isinstance(self.correction_enabled, bool):
            raise ConfigError("correction_enabled must be a bool")

    @classmethod
    def from_dict(cls, d: dict) -> "EngineConfig":
        allowed = set(cls.__dataclass_fields__)
        unknown = sorted(set(d) - allowed)
        if unknown:
            raise ConfigError(f"unknown config keys {unknown}; allowed keys are {sorted(allowed)}")
        return cls(**d)

    def to_dict(self) -> dict:
        return asdict(self)


@dataclass(frozen=True)
class StepTrace:
    step_index: int
    sim_time: float
    hit: bool
    candidate_len: int
    accepted_len: int
    lnew: int
    cache_alive_nodes: int
    event: str

    def to_dict(self) -> dict:
        return asdict(self)


@dataclass
class RunResult:
    output: list[TokenId]
    metrics: RunMetrics
    trace: list[StepTrace] = field(repr=False)
    wall: dict = field(default_factory=dict, repr=False)


def _check_pair(draft, target) -> None:
    if draft.vocab.size != target.vocab.size:
        raise ConfigError(f"draft and target vocabularies differ: {draft.vocab.size} vs {target.vocab.size}")
    if draft.eos_token != target.eos_token:
        raise ConfigError(f"draft and target disagree on the eos token: {draft.eos_token!r} vs {target.eos_token!r}")


def _check_prompt(prompt: Sequence[TokenId], vocab_size: int) -> list[TokenId]:
    toks = list(prompt)
    if not toks:
        raise InputError("prompt must contain at least one token")
    for i, t in enumerate(toks):
        if not isinstance(t, (int, np.integer)) or isinstance(t, bool) or t < 0 or t >= vocab_size:
            raise InputError(f"prompt token {t!r} at position {i} is out of vocabulary")
    return [int(t) for t in toks]


# ====================================================================== adapters
class _RowsAndTail:
    def __init__(self, rows_max: int, extra_max: int, order: int, dev):
        from .llama import RowBlock

        self.rows = RowBlock(rows_max, extra_max, dev)
        self.order = max(1, order)
        self.tail = torch.full((rows_max, self.order), -1, dtype=torch.int32, device=dev)

    def reset(self):
        self.rows.block.zero_()
        self.tail.fill_(-1)


class _KGramAdapter:
    """Device k-gram toy (lm.py:199-256 via card_kgram_dist)."""

    def __init__(self, model, rows_max: int, k: int, dev):
        self.m = model
        V = model.vocab.size
        self.V = V
        self.rows_max = rows_max
        self.k = k
        self.probs = torch.zeros((rows_max, V), dtype=torch.float64, device=dev)
        kk = min(k, V)
        self.kk = kk
        self.tok = torch.zeros((rows_max, k), dtype=torch.int32, device=dev)
        self.val = torch.zeros((rows_max, k), dtype=torch.float64, device=dev)
        self.cnt = torch.zeros(rows_max, dtype=torch.int32, device=dev)

    def reset(self):
        for t in (self.probs, self.tok, self.val, self.cnt):
            t.zero_()

    def _dists(self, rt: _RowsAndTail, t_score: float):
        m = self.m
        L_ = lib()
        M64 = (1 << 64) - 1
        off = rt.order - m.order   # the model reads context[-order:] (lm.py:235)
        tails = ctypes.c_void_p(rt.tail.data_ptr() + 4 * off)
        raise_for_status(L_.card_kgram_dist(m.seed & M64, m.mix_seed & M64, m.mix_weight, tails, m.order, rt.order,
                                            self.rows_max, self.V, m.sharpness, t_score, ptr(self.probs),
                                            stream_ptr()), "kgram_dist")
        if m.eos_token is not None:
            raise_for_status(L_.card_eos_fix(ptr(rt.rows.n_out), self.rows_max, ptr(rt.tail), rt.order, m.eos_token,
                                             self.V, ptr(self.probs), stream_ptr()), "eos_fix")

    def draft(self, run):
        self._dists(run.drt, run.t_score)
        L_ = lib()
        raise_for_status(L_.card_rows_topk(ptr(self.probs), self.rows_max, self.V, self.kk, ptr(self.tok),
                                           ptr(self.val), ptr(self.cnt), None, stream_ptr()), "rows_topk")
        return self.tok, self.val, self.cnt, 1

    def target(self, run):
        self._dists(run.trt, run.t_score)
        raise_for_status(lib().card_verify_probs(run.E_ptr, run.q_tok_ptr, ptr(self.probs), self.V, None,
                                                 ptr(run.uni), stream_ptr()), "verify_probs")

    def prefill(self, run, tokens):
        pass

    def post_correct(self, run):
        pass


class _LlamaAdapter:
    """Transformer draft/target (llama.py) with fused lm_head epilogues."""

    def __init__(self, model, role: str, run, rows_max: int):
        self.m = model
        self.role = role
        self.rows_max = rows_max
        tree_slots = run.cache_capacity if role == "draft" else 0
        budgets = {rows_max, PREFILL_CHUNK}
        dev = run.dev_d if role == "draft" else run.dev_t
        with torch.cuda.device(dev):
            if getattr(run, "private_runtimes", False):   # batched requests: own KV cache and buffers, shared weights
                from .llama import DeviceLlama

                self.rt = DeviceLlama(model.shard_cfg, model.packed, max_ctx=run.max_ctx, tree_slots=tree_slots,
                                      row_budgets=sorted(budgets), pool_requests=1)
            else:
                self.rt = model.runtime(run.max_ctx, tree_slots, budgets)
        if self.rt.dev != dev:
            raise ConfigError(f"the {role} model lives on {self.rt.dev}, the run places it on {dev}")
        if self.rt.extra_max < run.cfg.max_depth + 1:
            raise ConfigError("max_depth too large for the tree-attention extra-slot budget")
        # this request's prefix KV pages (returned to the runtime's pool with the adapter)
        with torch.cuda.device(dev):
            self.pages = self.rt.page_table(dev)
        V = model.vocab.size
        self.V = V
        self.k = run.cfg.k
        self.tok = torch.zeros((rows_max, self.k), dtype=torch.int32, device=dev)
        self.logp = torch.zeros((rows_max, self.k), dtype=torch.float64, device=dev)
        self.cnt = torch.zeros(rows_max, dtype=torch.int32, device=dev)
        self.amax = torch.zeros(rows_max, dtype=torch.int32, device=dev)
        self.lm_work = torch.zeros(lib().card_lmhead_work_floats(rows_max, self.k), dtype=torch.float32, device=dev)
        self.probs = torch.zeros((rows_max, V), dtype=torch.float64, device=dev) if run.sampling else None
        self.prefill_rows = None
        if role == "draft" and getattr(model, "fused_topk", False) and self.k <= 4:
            self.rt.lm_topk_head(rows_max)   # built before any graph capture
        if role == "draft":
            nL = model.cfg.n_layers
            row_bytes = self.rt.kv_row_elems() * self.rt.kv_esize()
            self.scratch_k = torch.zeros(run.cache_capacity * nL * row_bytes // 2, dtype=torch.int16, device=dev)
            self.scratch_v = torch.zeros_like(self.scratch_k)
            self.scratch_ptrs = torch.tensor([self.scratch_k.data_ptr(), self.scratch_v.data_ptr()],
                                             dtype=torch.int64, device=dev)

    def reset(self):
        """Per-request buffers back to their initial contents (session reuse)."""
        for t in (self.tok, self.logp, self.cnt, self.amax, self.lm_work, self.probs,
                  getattr(self, "scratch_k", None), getattr(self, "scratch_v", None)):
            if t is not None:
                t.zero_()

    def _bias_args(self, rt_tail: _RowsAndTail) -> tuple:
        """(ctx_tail, order, stride, seed, seed2, mix, sharpness) of the k-gram
        logit bias, applied on the fly by the top-k / argmax readers."""
        b = self.m.bias
        if b.sharpness == 0.0:
            return (None, 0, 0, 0, 0, 0.0, 0.0)
        M64 = (1 << 64) - 1
        tails = ctypes.c_void_p(rt_tail.tail.data_ptr() + 4 * (rt_tail.order - b.order))
        return (tails, b.order, rt_tail.order, b.seed & M64, b.mix_seed & M64, float(b.mix_weight),
                float(b.sharpness))

    def _bias(self, rt_tail: _RowsAndTail):
        """In-place bias of the logits (fp64 sampling path)."""
        tails, order, stride, seed, seed2, mix, sharp = self._bias_args(rt_tail)
        if sharp == 0.0:
            return
        raise_for_status(lib().card_logit_bias(ptr(self.rt.logits), ptr(rt_tail.rows.n_out), self.rows_max, self.V,
                                               tails, order, stride, seed, seed2, mix, sharp, stream_ptr()),
                         "logit_bias")

    def prefill(self, run, tokens):
        """Causal forward of tokens[0..n) into KV slots 0..n-1 (no outputs used)."""
        from .llama import RowBlock

        if not tokens:
            return
        if self.prefill_rows is None:
            self.prefill_rows = RowBlock(PREFILL_CHUNK, 1, self.rt.dev)
        nbytes = 0
        for s in range(0, len(tokens), PREFILL_CHUNK):
            chunk = tokens[s:s + PREFILL_CHUNK]
            nbytes += self.prefill_rows.set_chain(chunk, s, pages=self.pages)
            self.rt.forward(self.prefill_rows, PREFILL_CHUNK, pages=self.pages)
        return nbytes

    def _fused_lm_head(self):
        """The bf16 tcgen05 lm_head of the draft plan (None on the fp32 path)."""
        lm = self.rt.plans[self.rows_max].get("lm_head") if self.rt.fused else None
        return lm if lm is not None and lm.info["kind"] == 0 else None

    def _topk_head(self):
        """The fused lm_head + softmax + top-k linear (bf16 path, k <= 4) when
        the model asks for it (``LlamaModel.fused_topk``)."""
        if not getattr(self.m, "fused_topk", False) or self.k > 4:
            return None
        return self.rt.lm_topk_head(self.rows_max)

    def draft(self, run):
        rows = run.drt.rows
        bias = self._bias_args(run.drt)
        head = self._topk_head()
        if head is not None:
            # the lm_head epilogue reduces every 128-token vocab
            # tile to a top-4 + (max, sum-exp) record; no logits are stored
            L_ = lib()
            raise_for_status(L_.card_linear_fuse_kgram(head.h, *bias), "fuse_kgram")
            raise_for_status(L_.card_linear_fuse_topk(head.h, self.V, 1.0 / run.t_score), "fuse_topk")
            self.rt.forward(rows, self.rows_max, topk=True, pages=self.pages)
            raise_for_status(L_.card_lmhead_topk_merge(ptr(head.work), ptr(rows.n_out), self.rows_max, head.n_tiles,
                                                       self.k, self.V, ptr(self.tok), ptr(self.logp), ptr(self.cnt),
                                                       stream_ptr()), "lmhead_topk_merge")
            return self.tok, self.logp, self.cnt, 0
        lm = self._fused_lm_head() if bias[6] != 0.0 else None
        if lm is not None:
            # the k-gram bias rides in the lm_head epilogue (set for this launch
            # only: the plan is shared by every run of this model)
            raise_for_status(lib().card_linear_fuse_kgram(lm.h, *bias), "fuse_kgram")
        try:
            self.rt.forward(rows, self.rows_max, pages=self.pages)
        finally:
            if lm is not None:
                raise_for_status(lib().card_linear_fuse_kgram(lm.h, None, 0, 0, 0, 0, 0.0, 0.0), "fuse_kgram")
        if lm is not None:
            bias = (None, 0, 0, 0, 0, 0.0, 0.0)
        raise_for_status(lib().card_topk_logits(ptr(self.rt.logits), ptr(rows.n_out), self.rows_max, self.V, self.k,
                                                1.0 / run.t_score, ptr(self.tok), ptr(self.logp), ptr(self.cnt),
                                                ptr(self.lm_work), *bias, stream_ptr()),
                         "topk_logits")
        return self.tok, self.logp, self.cnt, 0

    def target(self, run):
        rows = run.trt.rows
        self.rt.forward(rows, self.rows_max, pages=self.pages)
        L_ = lib()
        if run.sampling:
            self._bias(run.trt)
            raise_for_status(L_.card_softmax64(ptr(self.rt.logits), ptr(rows.n_out), self.rows_max, self.V,
                                               1.0 / run.t_score, ptr(self.probs), stream_ptr()), "softmax64")
            raise_for_status(L_.card_verify_probs(run.E_ptr, run.q_tok_ptr, ptr(self.probs), self.V, None,
                                                  ptr(run.uni), stream_ptr()), "verify_probs")
        else:
            raise_for_status(L_.card_argmax_logits(ptr(self.rt.logits), ptr(rows.n_out), self.rows_max, self.V,
                                                   ptr(self.amax), ptr(self.lm_work), *self._bias_args(run.trt),
                                                   stream_ptr()), "argmax")
            raise_for_status(L_.card_verify_argmax(run.E_ptr, run.q_tok_ptr, ptr(self.amax), stream_ptr()),
                             "verify_argmax")

    def post_correct(self, run):
        """Draft KV roll-forward: promote accepted tree KV, then follow compaction."""
        if self.role != "draft":
            return
        rt = self.rt
        L_ = lib()
        nL = self.m.cfg.n_layers
        raise_for_status(L_.card_draft_promote(run.Ed_ptr, run.cache.handle, ptr(rt.k_ptrs), ptr(rt.v_ptrs), nL,
                                               rt.kv_row_elems(), rt.kv_esize(), rt.tree_base, run.cfg.max_depth + 2,
                                               _pt(self), stream_ptr()), "draft_promote")
        raise_for_status(L_.card_kv_compact(run.Ed_ptr, run.cache.handle, ptr(rt.k_ptrs), ptr(rt.v_ptrs), nL,
                                            rt.kv_row_elems(), rt.kv_esize(), rt.tree_base, ptr(self.scratch_ptrs),
                                            run.cache_capacity, stream_ptr()), "kv_compact")


def _pt(adapter):
    """Device page table of an adapter's request (None: identity / no KV)."""
    pages = getattr(adapter, "pages", None)
    return ptr(pages.dev) if pages is not None else None


def _adapter(model, role, run, rows_max):
    kind = getattr(model, "engine_kind", "host")
    if kind == "kgram":
        return _KGramAdapter(model, rows_max, run.cfg.k, run.dev)
    if kind == "llama":
        return _LlamaAdapter(model, role, run, rows_max)
    raise ConfigError(f"model kind {kind!r} has no device adapter (host-table models run via the TreeCache API)")


def _order_of(model) -> int:
    if getattr(model, "engine_kind", "") == "kgram":
        return model.order
    if getattr(model, "engine_kind", "") == "llama":
        return model.bias.order
    return 1


# ====================================================================== device run
class DeviceRun:
    """State of one decode on the device (engine.py:149-272)."""

    def __init__(self, draft, target, prompt, config: EngineConfig, *, trace_alive: bool = True,
                 devices: tuple[int, int] | None = None, private_runtimes: bool = False):
        _check_pair(draft, target)
        self.private_runtimes = private_runtimes
        self.draft_model, self.target_model = draft, target
        self.cfg = config
        self.dev = require_cuda()
        # placement (mode="concurrent"): the candidate tree, the draft state and
        # the draft rows live with the draft model; committed tokens, the target
        # state and rows with the target.  Kernels of either side read the other
        # side's small buffers (query result, commit outcome, committed tokens)
        # directly — over NVLink P2P when the devices differ.
        dd, td = devices if devices is not None else (self.dev.index, self.dev.index)
        self.dev_d, self.dev_t = torch.device("cuda", dd), torch.device("cuda", td)
        if dd != td:
            enable_peer_access(dd, td)
        self.prompt = _check_prompt(prompt, target.vocab.size)
        self.t_score = config.temperature if config.temperature > 0.0 else 1.0
        self.sampling = config.temperature > 0.0
        self.trace_alive = trace_alive
        self.eos = target.eos_token
        cfg = config
        C0 = len(self.prompt)
        self.max_ctx = C0 + cfg.max_new_tokens + cfg.max_depth + 8
        if cfg.correction_enabled:
            self.cache_capacity = 6 * cfg.K * (cfg.max_depth + 1) + 256
        else:   # the un-steered ablation never compacts (cache.py:415-437)
            self.cache_capacity = cfg.K * (cfg.max_new_tokens + cfg.max_depth + 2) * 2 + 256
        with torch.cuda.device(self.dev_d):
            self.cache = TreeCache(self.prompt[-1], CacheConfig(cfg.K, cfg.k, cfg.max_depth), eos_token=self.eos,
                                   capacity=self.cache_capacity)
        order = max(_order_of(draft), _order_of(target))
        self.d_rows_max = cfg.K + cfg.max_depth + 2
        self.t_rows_max = cfg.query_depth + 1
        self.drt = _RowsAndTail(self.d_rows_max, cfg.max_depth + 1, order, self.dev_d)
        self.trt = _RowsAndTail(self.t_rows_max, 1, order, self.dev_t)
        self.committed = torch.zeros(self.max_ctx + 8, dtype=torch.int32, device=self.dev_t)
        self.committed[:C0] = torch.tensor(self.prompt, dtype=torch.int32)
        # host<->device bytes of the current request (the bench's e2e record)
        self.io = {"h2d": 4 * C0, "d2h": 0}
        rng = np.random.default_rng(cfg.seed)   # engine.py:162; the only randomness
        n_uni = (cfg.max_new_tokens + 2) * (cfg.query_depth + 2) + 16 if self.sampling else 1
        self.uni = torch.from_numpy(rng.random(n_uni)).to(self.dev_t)
        st = EngineState()
        st.C = C0
        st.Pd = 0
        st.max_new = cfg.max_new_tokens
        st.eos = -1 if self.eos is None else int(self.eos)
        st.order = order
        st.sampling = int(self.sampling)
        st.base_len = C0
        st.anchor_origin = int(not cfg.correction_enabled)
        st.n_uni = n_uni
        self.E = torch.frombuffer(bytearray(bytes(st)), dtype=torch.int32).to(self.dev_t)
        self.io["h2d"] += self.uni.numel() * 8 + self.E.numel() * 4
        self._E0 = self.E.clone()   # initial state, for rebind()
        self.E_ptr = ptr(self.E)
        # draft-side state: the same buffer in the lockstep drivers; a separate
        # copy in mode="concurrent" (the draft stream never reads the target's
        # in-flight commit; card_engine_handoff passes it over after each verify)
        self.concurrent = config.mode == "concurrent"
        if dd != td and not self.concurrent:
            raise ConfigError("separate draft/target devices need mode='concurrent'")
        self.Ed = self.E.to(self.dev_d, copy=True) if self.concurrent else self.E
        self.Ed_ptr = ptr(self.Ed)
        self.q_tok_ptr = ctypes.c_void_p(self.cache._qbufs[1])
        self._host = torch.empty(self.E.numel(), dtype=torch.int32, pin_memory=True)
        self._host_d = torch.empty(self.E.numel(), dtype=torch.int32, pin_memory=True)
        self.da = _adapter(draft, "draft", self, self.d_rows_max)
        self.ta = _adapter(target, "target", self, self.t_rows_max)
        self._field = {name: getattr(EngineState, name).offset // 4 for name, _ in EngineState._fields_}
        self.output: list[int] = []
        self.trace: list[StepTrace] = []
        self.graphs = None
        self.timing = {}

    def rebind(self, prompt) -> None:
        """Start a new request on this run's device buffers, keeping its
        captured graphs (which point into them).  The prompt length and the
        config must be the ones the run was built for; every buffer the first
        step could read is restored to its constructor contents."""
        prompt = _check_prompt(prompt, self.target_model.vocab.size)
        if len(prompt) != len(self.prompt):
            raise ConfigError("rebind needs a prompt of the run's length")
        self.prompt = prompt
        C0 = len(prompt)
        with torch.cuda.device(self.dev_d):
            self.cache.clear(prompt[-1])
        self.committed.zero_()
        self.committed[:C0] = torch.tensor(prompt, dtype=torch.int32)
        self.io = {"h2d": 4 * C0, "d2h": 0}
        self.E.copy_(self._E0)
        if self.Ed is not self.E:
            self.Ed.copy_(self._E0)
        self.drt.reset()
        self.trt.reset()
        self.da.reset()
        self.ta.reset()
        self.output = []
        self.trace = []
        self.timing = {}
        if self.graphs is not None:
            self.replays = [0, 0]

    # ---------------------------------------------------------------- state io
    def _fptr(self, name: str, draft: bool = False) -> ctypes.c_void_p:
        buf = self.Ed if draft else self.E
        return ctypes.c_void_p(buf.data_ptr() + 4 * self._field[name])

    def read_state(self) -> EngineState:
        self._host.copy_(self.E, non_blocking=True)
        self.io["d2h"] += self.E.numel() * 4
        torch.cuda.current_stream().synchronize()
        return EngineState.from_buffer_copy(self._host.numpy().tobytes())

    def _set_field(self, name: str, value: int):
        self.E[self._field[name]] = int(value)
        self.io["h2d"] += 4
        if self.Ed is not self.E:
            self.Ed[self._field[name]] = int(value)
            self.io["h2d"] += 4

    def prefill(self):
        """Prompt KV for both models: target gets prompt[:-1] (its last token is
        the first verify input), the draft likewise (its flat step computes the root)."""
        body = self.prompt[:-1]
        with torch.cuda.device(self.dev_d):
            self.io["h2d"] += self.da.prefill(self, body) or 0
        with torch.cuda.device(self.dev_t):
            self.io["h2d"] += self.ta.prefill(self, body) or 0
        self._set_field("Pd", len(body))

    # ---------------------------------------------------------------- sequences
    def launch_draft_step(self):
        L_ = lib()
        s = stream_ptr()
        raise_for_status(L_.card_draft_rows(self.Ed_ptr, self.cache.handle, ptr(self.committed), ptr(self.drt.rows.block),
                                            self.d_rows_max, self.drt.rows.extra_max,
                                            getattr(self.da, "rt", None).tree_base if hasattr(self.da, "rt") else 0,
                                            ptr(self.drt.tail), self.drt.order, _pt(self.da), s), "draft_rows")
        tok, val, cnt, probs = self.da.draft(self)
        raise_for_status(L_.card_cache_expand_topk(self.cache.handle, ptr(tok), ptr(val), ptr(cnt), -1, probs,
                                                   self._fptr("stop", True), s), "expand")
        raise_for_status(L_.card_record_width(self.Ed_ptr, self.cache.handle, ptr(self.drt.rows.n_out), s), "record")

    def launch_target_step(self, with_correct: bool = True, readback: bool = True, with_query: bool = True):
        L_ = lib()
        s = stream_ptr()
        if with_query:
            raise_for_status(L_.card_cache_query(self.cache.handle, self.cfg.query_depth, s), "query")
        raise_for_status(L_.card_target_rows(self.E_ptr, self.cache.handle, ptr(self.committed),
                                             ptr(self.trt.rows.block), self.t_rows_max, 1, ptr(self.trt.tail),
                                             self.trt.order, _pt(self.ta), s), "target_rows")
        self.ta.target(self)
        raise_for_status(L_.card_commit(self.E_ptr, ptr(self.committed), s), "commit")
        if with_correct:
            self.launch_correct()
        raise_for_status(L_.card_cycle_end(self.E_ptr, None if self.concurrent else self.cache.handle, s),
                         "cycle_end")
        if readback:
            self._host.copy_(self.E, non_blocking=True)
            self.io["d2h"] += self.E.numel() * 4

    # ---------------------------------------------------------------- helpers
    def _alive(self) -> int:
        if not self.trace_alive:
            return -1
        return self.cache.alive_below_root()

    def _emit(self, t, hit, cl, al, ln, ev):
        self.trace.append(StepTrace(len(self.trace), t, bool(hit), int(cl), int(al), int(ln), self._alive(), ev))

    def _check_cache_status(self):
        st = self.cache.state()
        if st.status not in (0, -4):
            raise_for_status(st.status, "device cache")

    # ---------------------------------------------------------------- stepwise driver
    def draft_step_sync(self) -> int:
        self.launch_draft_step()
        E = self.read_state()
        self._check_cache_status()
        w = E.widths[E.n_widths - 1] if 0 < E.n_widths <= 64 else 0
        self._set_field("stop", 0)
        self._set_field("n_widths", 0)
        return w

    def target_step_sync(self):
        self.launch_target_step(with_correct=False, readback=False)
        E = self.read_state()
        self._check_cache_status()
        return E

    def launch_correct(self):
        L_ = lib()
        s = stream_ptr()
        raise_for_status(L_.card_cache_correct(self.cache.handle, self._fptr("acc", True), self._fptr("n_acc", True),
                                               self._fptr("corr", True), self._fptr("done", True), s), "correct")
        self.da.post_correct(self)

    def correct_sync(self):
        self.launch_correct()
        torch.cuda.current_stream().synchronize()
        self._check_cache_status()

    def run_stepwise(self):
        """_run_serial (engine.py:290-317) with one host sync per step."""
        cfg = self.cfg
        d_lat = self.draft_model.spec.forward_latency
        t_lat = self.target_model.spec.forward_latency
        self.prefill()
        clock = 0.0
        for _ in range(cfg.query_depth):
            w = self.draft_step_sync()
            if w == 0:
                break
            clock += d_lat
            self._emit(clock, False, w, 0, 0, "draft_expand")
        done = False
        while not done:
            start, n_exp = clock, 0
            for _ in range(cfg.ratio):
                w = self.draft_step_sync()
                if w == 0:
                    break
                n_exp += 1
                self._emit(start + n_exp * d_lat, False, w, 0, 0, "draft_expand")
            E = self.target_step_sync()
            clock = start + max(n_exp * d_lat, t_lat)
            hit = bool(E.rec_hit)
            self.output.extend(E.committed_now[i] for i in range(E.n_commit))
            if cfg.correction_enabled:
                self._emit_target(clock, hit, E)
                done = bool(E.done)
                if not done:
                    self.correct_sync()
                    self._emit(clock, hit, 0, 0, 0, "correct")
            else:
                done = bool(E.done)
                self._emit_target(clock, hit, E, alive_before_update=True)
                if not done:
                    self._ablation_update(E)
                    self._emit(clock, hit, 0, 0, 0, "correct")

    def _emit_target(self, clock, hit, E, alive_before_update=False):
        self._emit(clock, hit, E.rec_L if hit else 0, E.rec_acc, E.rec_lnew, "verify" if hit else "miss_step")

    def _ablation_update(self, E):
        """engine.py:269-272: advance_root, else reset to the last output."""
        n = E.rec_n_acc
        acc = [E.acc[i] for i in range(n)]
        moved = self.cache.advance_root(acc, E.rec_corr)
        if not moved:
            self.cache.reset(self.output[-1])
            C = len(self.prompt) + len(self.output)
            self._set_field("base_len", C)

    # ---------------------------------------------------------------- graph driver
    def capture(self):
        """Capture one draft step and one target step as CUDA graphs."""
        if not self.cfg.correction_enabled:
            raise ConfigError("graph mode needs correction_enabled=True (the ablation resets on the host)")
        from . import _lib

        g_d, g_t = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        # capture records without executing: the run state is untouched
        with torch.cuda.stream(s):
            c0 = _lib.launch_count[0]
            with torch.cuda.graph(g_d, stream=s):
                self.launch_draft_step()
            c1 = _lib.launch_count[0]
            with torch.cuda.graph(g_t, stream=s):
                self.launch_target_step(with_correct=True, readback=True)
            c2 = _lib.launch_count[0]
        torch.cuda.current_stream().wait_stream(s)
        self.graphs = (g_d, g_t)
        self.launches_per_graph = (c1 - c0, c2 - c1)
        self.replays = [0, 0]

    def graph_cycles(self, max_cycles: int | None = None):
        """The graph driver as a generator (engine.py:290-317 schedule): each
        step launches work on the current stream, records an event and yields
        it; the caller resumes it once the event has completed.  One
        host<->device round trip per cycle; run_graphs() drives one request,
        the batch driver interleaves several on their own streams."""
        cfg = self.cfg
        d_lat = self.draft_model.spec.forward_latency
        t_lat = self.target_model.spec.forward_latency
        g_d, g_t = self.graphs
        clock = 0.0
        depth = 0
        for _ in range(cfg.query_depth):   # warm-up (engine.py:295-301)
            g_d.replay()
            self.replays[0] += 1
        self._host.copy_(self.E, non_blocking=True)
        self.io["d2h"] += self.E.numel() * 4
        ev = torch.cuda.Event()
        ev.record()
        yield ev
        E = EngineState.from_buffer_copy(self._host.numpy().tobytes())
        for i in range(min(E.n_widths, 64)):
            w = E.widths[i]
            if w == 0:
                break
            depth += 1
            clock += d_lat
            self._emit(clock, False, w, 0, 0, "draft_expand")
        self._set_field("n_widths", 0)
        self._set_field("stop", 0)
        done = False
        cycles = 0
        while not done:
            n_exp = min(cfg.ratio, max(0, cfg.max_depth - depth))
            for _ in range(n_exp):
                g_d.replay()
            g_t.replay()   # ends with the record copy into self._host
            self.io["d2h"] += self.E.numel() * 4
            self.replays[0] += n_exp
            self.replays[1] += 1
            ev = torch.cuda.Event()
            ev.record()
            yield ev
            E = EngineState.from_buffer_copy(self._host.numpy().tobytes())
            start, k = clock, 0
            for i in range(min(E.rec_n_widths, 64)):
                w = E.rec_widths[i]
                if w == 0:
                    break
                k += 1
                self._emit(start + k * d_lat, False, w, 0, 0, "draft_expand")
            clock = start + max(k * d_lat, t_lat)
            hit = bool(E.rec_hit)
            self.output.extend(E.committed_now[i] for i in range(E.n_commit))
            self._emit_target(clock, hit, E)
            done = bool(E.rec_done)
            if not done:
                self._emit(clock, hit, 0, 0, 0, "correct")
            depth = E.rec_depth
            cycles += 1
            if max_cycles is not None and cycles >= max_cycles:
                break
        self.cycles = cycles

    def run_graphs(self, max_cycles: int | None = None):
        """Throughput driver: one host<->device round trip per cycle."""
        for ev in self.graph_cycles(max_cycles):
            ev.synchronize()
        return self.cycles


_GREEN: dict = {}
_DRAFT_PRIORITY = -8   # concurrent mode, shared SMs: the draft stream first (clamped to the highest priority)


def _green_partition(device: int, draft_sms: int):
    """The (draft, target) SM partitions of one GPU (card_green) as stream
    pointers and SM counts, created once per process and split: graphs
    captured on the streams keep referring to them, so they live as long
    as the process."""
    key = (device, draft_sms)
    if key not in _GREEN:
        g = ctypes.c_void_p()
        raise_for_status(lib().card_green_create(device, draft_sms, ctypes.byref(g)), "card_green_create")
        ptrs, sms = [], []
        for part in (0, 1):
            sp, n = ctypes.c_void_p(), ctypes.c_int()
            raise_for_status(lib().card_green_stream(g, part, ctypes.byref(sp), ctypes.byref(n)), "card_green_stream")
            ptrs.append(sp.value)
            sms.append(n.value)
        _GREEN[key] = (g, ptrs, sms)
    return _GREEN[key][1], _GREEN[key][2]


class _ConcurrentDriver:
    """mode="concurrent" (engine.py:320-389) on one GPU: the draft expands the
    tree on its own stream while the target verifies on another.  The
    reference's lock + epoch protocol becomes stream order plus a hand-off:

      draft stream  : [draft step]* ... wait(V) [handoff E->Ed, correct,
                      draft-KV roll-forward, query] -> event Q ... [draft step]*
      target stream : wait(Q) [target rows, verify forward, accept, commit,
                      record -> host] -> event V

    The cache is only mutated on the draft stream, so corrections and
    expansions never race (the reference discards stale expansions by epoch,
    engine.py:359-360; here they are ordered).  At most one draft step is in
    flight so a correction waits for at most one.  Greedy output is
    schedule-invariant (lossless); the trace carries wall-clock times."""

    def _streams(self, run: "DeviceRun", draft_sms: int | None):
        """The draft and target streams.  draft_sms (one GPU): two SM
        partitions (card_green), the draft's persistent forward sized to its
        share; otherwise two streams sharing every SM, the draft's at the
        higher priority (with the target verifying concurrently, accepted
        tokens per second track draft layers per second)."""
        dd, td = run.dev_d, run.dev_t
        self.green = None
        self.draft_sms = None
        if draft_sms:
            if dd != td:
                raise ConfigError("draft_sms partitions one GPU; the draft and target are on two")
            ptrs, sms = _green_partition(dd.index, int(draft_sms))
            self.draft_sms, self.target_sms = sms
            self.D = torch.cuda.ExternalStream(ptrs[0], device=dd)
            self.T = torch.cuda.ExternalStream(ptrs[1], device=td)
        else:
            self.D = torch.cuda.Stream(device=dd, priority=_DRAFT_PRIORITY)
            self.T = torch.cuda.Stream(device=td, priority=0)

    def _capture_fn(self, counter):
        """capture(graph, device, fn): on the side's own stream (a graph keeps
        the SM partition of the stream it was captured on); the draft's
        persistent forward sized to the partition while capturing."""
        from . import _lib

        def capture(g, dev, fn):
            side = self.D if dev == self.run.dev_d else self.T
            pf = [p["pfwd"] for p in getattr(getattr(self.run.da, "rt", None), "plans", {}).values() if "pfwd" in p] \
                if (self.draft_sms and side is self.D) else []
            for f in pf:
                raise_for_status(lib().card_pfwd_set_grid(f.h, self.draft_sms), "card_pfwd_set_grid")
            try:
                with torch.cuda.device(dev):
                    side.wait_stream(torch.cuda.current_stream(dev))
                    with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
                        fn()
                    torch.cuda.current_stream(dev).wait_stream(side)
            finally:
                for f in pf:   # the serial drivers keep the whole device
                    lib().card_pfwd_set_grid(f.h, 0)
            counter.append(_lib.launch_count[0])
        return capture

    def __del__(self):
        pass

    def __init__(self, run: "DeviceRun", draft_sms: int | None = None):
        from . import _lib

        self.run = run
        dd, td = run.dev_d, run.dev_t
        run.q_tok_ptr = ctypes.c_void_p(run.cache._qbufs[1])   # the verify reads the cache's query buffer
        self._streams(run, draft_sms)
        self.g_d, self.g_q, self.g_t, self.g_c = (torch.cuda.CUDAGraph() for _ in range(4))
        c = [_lib.launch_count[0]]
        capture = self._capture_fn(c)

        def draft_step():
            run.launch_draft_step()
            run._host_d.copy_(run.Ed, non_blocking=True)

        def query():
            raise_for_status(lib().card_cache_query(run.cache.handle, run.cfg.query_depth, stream_ptr()), "query")

        def correct_query():
            raise_for_status(lib().card_engine_handoff(run.E_ptr, run.Ed_ptr, stream_ptr()), "handoff")
            run.launch_correct()
            query()

        capture(self.g_d, dd, draft_step)
        capture(self.g_q, dd, query)
        capture(self.g_t, td, lambda: run.launch_target_step(with_correct=False, readback=True, with_query=False))
        capture(self.g_c, dd, correct_query)
        self.per_graph = [c[i + 1] - c[i] for i in range(4)]
        self.replays = [0, 0, 0, 0]

    def _draft(self):
        with torch.cuda.stream(self.D):
            self.g_d.replay()
            ev = torch.cuda.Event()
            ev.record(self.D)
        self.replays[0] += 1
        self.run.io["d2h"] += self.run.Ed.numel() * 4   # the captured width-record readback
        return ev

    def _now(self, t0) -> float:
        """Trace clock in latency units: wall seconds / time_scale, as the
        reference's concurrent mode stamps its events (engine.py:330-331)."""
        return (time.perf_counter() - t0) / self.run.cfg.time_scale

    def _draft_done(self, t0):
        """Read the finished draft step's record: width (trace) and stop flag."""
        run = self.run
        Ed = EngineState.from_buffer_copy(run._host_d.numpy().tobytes())
        n = Ed.n_widths
        w = Ed.widths[n - 1] if 0 < n <= 64 else 0
        if w > 0:
            run._emit(self._now(t0), False, w, 0, 0, "draft_expand")
        return bool(Ed.stop)

    def run_loop(self):
        run, cfg = self.run, self.run.cfg
        t0 = time.perf_counter()
        for dev, st in ((run.dev_d, self.D), (run.dev_t, self.T)):
            torch.cuda.current_stream(dev).synchronize()
            st.wait_stream(torch.cuda.current_stream(dev))
        # warm-up: query_depth expansions before the first target step (engine.py:377)
        paused = False
        for _ in range(min(cfg.query_depth, cfg.max_depth)):
            ev = self._draft()
            ev.synchronize()
            if self._draft_done(t0):
                paused = True
                break
        with torch.cuda.stream(self.D):
            self.g_q.replay()
            q_ev = torch.cuda.Event()
            q_ev.record(self.D)
        self.replays[1] += 1
        d_ev = None
        done = False
        while not done:
            self.T.wait_event(q_ev)
            with torch.cuda.stream(self.T):
                self.g_t.replay()
                v_ev = torch.cuda.Event()
                v_ev.record(self.T)
            self.replays[2] += 1
            run.io["d2h"] += run.E.numel() * 4
            while not v_ev.query():
                if d_ev is not None and d_ev.query():
                    paused = self._draft_done(t0)
                    d_ev = None
                if d_ev is None and not paused:
                    d_ev = self._draft()
            E = EngineState.from_buffer_copy(run._host.numpy().tobytes())
            now = self._now(t0)
            hit = bool(E.rec_hit)
            run.output.extend(E.committed_now[i] for i in range(E.n_commit))
            run._emit_target(now, hit, E)
            done = bool(E.rec_done)
            if done:
                break
            if d_ev is not None:   # the correction follows the in-flight draft step on its stream
                d_ev.synchronize()
                self._draft_done(t0)
                d_ev = None
            self.D.wait_event(v_ev)
            with torch.cuda.stream(self.D):
                self.g_c.replay()
                q_ev = torch.cuda.Event()
                q_ev.record(self.D)
            self.replays[3] += 1
            paused = False
            run._emit(self._now(t0), hit, 0, 0, 0, "correct")
        for dev in {run.dev_d, run.dev_t}:
            torch.cuda.synchronize(dev)

    def launches(self) -> int:
        return sum(r * n for r, n in zip(self.replays, self.per_graph))


class _MailboxDriver(_ConcurrentDriver):
    """mode="concurrent" with the exchange in device mailboxes
    (csrc/card_mailbox.cu): the default when the draft and
    the target live on two GPUs.  Neither side waits on the host or on the
    other's stream: the target's verify graph opens with a kernel that
    blocks on the query box (an acquire poll on memory the draft GPU writes
    with P2P stores and a system-scope release), and every draft step opens
    with a non-blocking poll of the commit box, then corrects the tree,
    queries it and publishes the query before it expands.  The tree is
    mutated only by the draft stream, so an expansion always follows the
    latest correction it has seen (the reference's epoch check,
    engine.py:359-360, can never fire); the epoch rides along with each
    query.  The host only keeps one draft step in flight, relaunches the
    verify graph and reads the records for the trace."""

    def __init__(self, run: "DeviceRun", draft_sms: int | None = None):
        from . import _lib

        self.run = run
        dd, td = run.dev_d, run.dev_t
        rt = getattr(run.da, "rt", None)
        if dd == td and draft_sms:
            # measured: graphs on the two green-context streams did not run
            # side by side, so the verify graph's blocking wait starved the draft
            raise ConfigError("exchange='mailbox' does not run on SM partitions of one GPU; use exchange='events'")
        if dd == td and rt is not None and any("pfwd" in p for p in rt.plans.values()):
            # the target's verify graph blocks on the query box while the draft's
            # persistent forward needs every SM (cooperative launch): on one GPU
            # the two would wait for each other
            raise ConfigError("exchange='mailbox' on one GPU needs a draft without the persistent forward "
                              "(LlamaModel(persistent=False)); or exchange='events' or two GPUs")
        L_ = lib()
        h = ctypes.c_void_p()
        raise_for_status(L_.card_mailbox_create(dd.index, td.index, ctypes.byref(h)), "card_mailbox_create")
        self.mb = h
        skip = ctypes.c_void_p()
        L_.card_mailbox_skip_flag(h, ctypes.byref(skip))
        view, q_tok = ctypes.c_void_p(), ctypes.c_void_p()
        L_.card_mailbox_query_view(h, ctypes.byref(view), ctypes.byref(q_tok))
        self.skip, self.view = skip, view
        run.q_tok_ptr = q_tok   # the verify reads the delivered candidate tokens
        self._streams(run, draft_sms)
        self.g_d, self.g_q, self.g_t, self.g_c = (torch.cuda.CUDAGraph() for _ in range(4))
        c = [_lib.launch_count[0]]
        capture = self._capture_fn(c)

        cache = run.cache.handle

        def exchange():   # the draft side of one exchange: poll, correct, query, publish (all gated)
            s = stream_ptr()
            raise_for_status(L_.card_mailbox_poll_commit(h, run.Ed_ptr, s), "poll_commit")
            raise_for_status(L_.card_cache_correct(cache, run._fptr("acc", True), run._fptr("n_acc", True),
                                                   run._fptr("corr", True), skip, s), "correct")
            run.da.post_correct(run)
            raise_for_status(L_.card_cache_query_if(cache, run.cfg.query_depth, skip, s), "query_if")
            raise_for_status(L_.card_mailbox_publish_query(h, cache, 0, s), "publish_query")

        def draft_step():
            exchange()
            run.launch_draft_step()
            run._host_d.copy_(run.Ed, non_blocking=True)

        def exchange_only():
            exchange()
            run._host_d.copy_(run.Ed, non_blocking=True)

        def first_query():
            s = stream_ptr()
            raise_for_status(L_.card_cache_query(cache, run.cfg.query_depth, s), "query")
            raise_for_status(L_.card_mailbox_publish_query(h, cache, 1, s), "publish_query")

        def target_step():
            s = stream_ptr()
            raise_for_status(L_.card_mailbox_wait_query(h, s), "wait_query")
            raise_for_status(L_.card_target_rows_view(run.E_ptr, view, q_tok, ptr(run.committed),
                                                      ptr(run.trt.rows.block), run.t_rows_max, 1, ptr(run.trt.tail),
                                                      run.trt.order, _pt(run.ta), s), "target_rows_view")
            run.ta.target(run)
            raise_for_status(L_.card_commit(run.E_ptr, ptr(run.committed), s), "commit")
            raise_for_status(L_.card_mailbox_publish_commit(h, run.E_ptr, s), "publish_commit")
            raise_for_status(L_.card_cycle_end(run.E_ptr, None, s), "cycle_end")
            run._host.copy_(run.E, non_blocking=True)

        capture(self.g_d, dd, draft_step)
        capture(self.g_q, dd, first_query)
        capture(self.g_t, td, target_step)
        capture(self.g_c, dd, exchange_only)
        self.per_graph = [c[i + 1] - c[i] for i in range(4)]
        self.replays = [0, 0, 0, 0]

    def __del__(self):
        try:
            lib().card_mailbox_destroy(self.mb)
        except Exception:
            pass

    def _exchange(self):
        with torch.cuda.stream(self.D):
            self.g_c.replay()
            ev = torch.cuda.Event()
            ev.record(self.D)
        self.replays[3] += 1
        self.run.io["d2h"] += self.run.Ed.numel() * 4
        return ev

    def run_loop(self):
        run, cfg = self.run, self.run.cfg
        t0 = time.perf_counter()
        for dev, st in ((run.dev_d, self.D), (run.dev_t, self.T)):
            torch.cuda.current_stream(dev).synchronize()
            st.wait_stream(torch.cuda.current_stream(dev))
        # a previous request may have left a commit / query unread
        raise_for_status(lib().card_mailbox_reset(self.mb), "card_mailbox_reset")
        paused = False
        for _ in range(min(cfg.query_depth, cfg.max_depth)):   # warm-up (engine.py:377)
            ev = self._draft()
            ev.synchronize()
            if self._draft_done(t0):
                paused = True
                break
        with torch.cuda.stream(self.D):
            self.g_q.replay()
        self.replays[1] += 1
        d_ev = None
        while True:
            with torch.cuda.stream(self.T):
                self.g_t.replay()   # blocks on the device until the next query arrives
                v_ev = torch.cuda.Event()
                v_ev.record(self.T)
            self.replays[2] += 1
            run.io["d2h"] += run.E.numel() * 4
            while not v_ev.query():
                if d_ev is not None and d_ev.query():
                    paused = self._draft_done(t0)
                    d_ev = None
                if d_ev is None:   # a paused draft still polls, corrects and publishes
                    d_ev = self._exchange() if paused else self._draft()
            E = EngineState.from_buffer_copy(run._host.numpy().tobytes())
            hit = bool(E.rec_hit)
            run.output.extend(E.committed_now[i] for i in range(E.n_commit))
            run._emit_target(self._now(t0), hit, E)
            if E.rec_done:
                break
            run._emit(self._now(t0), hit, 0, 0, 0, "correct")
        if d_ev is not None:
            d_ev.synchronize()
        for dev in {run.dev_d, run.dev_t}:
            torch.cuda.synchronize(dev)


def _validate_run_config(draft, target, config):
    """Limits of the device engine only (host-table pairs run the reference
    algorithm on the host and take any depth): the engine state keeps 64
    accepted tokens per verify (card_engine_state.acc), and the transformer
    tree attention gathers at most 31 ancestor slots per row."""
    kinds = {getattr(draft, "engine_kind", "host"), getattr(target, "engine_kind", "host")}
    if "host" in kinds:
        return
    if config.query_depth > 62:
        raise ConfigError(f"query_depth {config.query_depth} > 62: the device engine state holds 64 accepted tokens")
    if "llama" in kinds and config.max_depth > 30:
        raise ConfigError(f"max_depth {config.max_depth} > 30 is not supported by the device tree attention")


def enable_peer_access(a: int, b: int):
    """P2P loads/stores between two devices in both directions (NVLink)."""
    raise_for_status(lib().card_enable_peer_access(a, b), "card_enable_peer_access")


_SESSIONS_PER_TARGET = 2


def _model_sig(model) -> tuple:
    """What a captured run depends on besides the weights: identity, EOS and
    the agreement-bias / k-gram parameters (all baked into the graphs)."""
    fields = ("eos_token", "bias", "seed", "mix_seed", "mix_weight", "sharpness", "order", "fused_topk")
    return (id(model),) + tuple(repr(getattr(model, f, None)) for f in fields)


def _session_run(draft, target, prompt, config: EngineConfig, trace_alive: bool,
                 devices: tuple[int, int] | None = None) -> DeviceRun:
    """A serving session per (draft, target, config, prompt length): the run's
    device buffers and its two captured graphs are built by the first request
    and reused by the next ones (rebind), as a server captures its graphs
    once per shape at start-up.  Kept on the target model, at most
    _SESSIONS_PER_TARGET of them, least recently used dropped first."""
    key = (_model_sig(draft), _model_sig(target), len(prompt), tuple(sorted(config.to_dict().items())),
           bool(trace_alive), devices)
    store = target.__dict__.setdefault("_card_sessions", {})
    run = store.pop(key, None)
    if run is not None and run.draft_model is draft:
        run.rebind(prompt)
    else:
        run = DeviceRun(draft, target, prompt, config, trace_alive=trace_alive, devices=devices)
    store[key] = run
    while len(store) > _SESSIONS_PER_TARGET:
        store.pop(next(iter(store)))
    return run


def run_speculative(draft, target, prompt: Sequence[TokenId], config: EngineConfig, *,
                    use_graphs: bool | None = None, trace_alive: bool | None = None,
                    devices: tuple[int, int] | None = None, exchange: str | None = None,
                    draft_sms: int | None = None) -> RunResult:
    """The generate() entry point (engine.py:275-287), on the device.

    mode="concurrent": ``exchange`` picks how draft and target hand over
    queries and corrections — "mailbox" (device mailboxes, the default when
    ``devices`` puts them on two GPUs) or "events" (stream events and a host
    hand-off, the default on one GPU).  ``draft_sms`` (one GPU) splits the
    SMs into a draft partition of that many SMs and a target partition, so
    the latency-bound draft steps and the bandwidth-bound verify overlap.

    ``use_graphs`` (default: True for transformer pairs with correction on)
    selects the CUDA-graph driver; the stepwise driver reproduces the
    reference trace exactly, including ``cache_alive_nodes``."""
    _validate_run_config(draft, target, config)
    kinds = {getattr(draft, "engine_kind", "host"), getattr(target, "engine_kind", "host")}
    if "host" in kinds:
        from .hostrun import run_host_models

        return run_host_models(draft, target, prompt, config)
    if use_graphs is None:
        # a tensor-parallel target's collectives go through torch.distributed
        # (NCCL or gloo) and run eagerly: the stepwise driver
        tp = getattr(target, "tp", None) is not None or getattr(draft, "tp", None) is not None
        use_graphs = "llama" in kinds and config.correction_enabled and not tp
    if trace_alive is None:
        trace_alive = not use_graphs
    concurrent = config.mode == "concurrent" and config.correction_enabled and use_graphs
    if devices is not None and not concurrent:
        raise ConfigError("devices=(draft, target) placement needs mode='concurrent' with a transformer pair")
    if concurrent:
        run = _session_run(draft, target, prompt, config, False, devices=devices)
        t0 = time.perf_counter()
        run.prefill()
        if exchange is None:
            exchange = "mailbox" if run.dev_d != run.dev_t else "events"
        if exchange not in ("mailbox", "events"):
            raise ConfigError(f"exchange must be 'mailbox' or 'events', got {exchange!r}")
        drv = getattr(run, "_cdriver", None)
        kind = _MailboxDriver if exchange == "mailbox" else _ConcurrentDriver
        if type(drv) is not kind or drv.draft_sms_req != draft_sms:   # captured once per session and setup
            run._cdriver = None
            drv = run._cdriver = kind(run, draft_sms)
            drv.draft_sms_req = draft_sms
        drv.replays = [0, 0, 0, 0]
        for dev in {run.dev_d, run.dev_t}:
            torch.cuda.synchronize(dev)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev0.record(torch.cuda.current_stream(run.dev_t))
        drv.run_loop()   # ends with both devices synchronised
        ev1 = torch.cuda.Event(enable_timing=True)
        ev1.record(torch.cuda.current_stream(run.dev_t))
        ev1.synchronize()
        run.timing["decode_ms"] = ev0.elapsed_time(ev1)
        run.timing["gpu_launches"] = drv.launches()
        run.timing["draft_steps"], run.timing["target_steps"] = drv.replays[0], drv.replays[2]
        run.timing["wall_s"] = time.perf_counter() - t0
        run.timing["h2d_bytes"], run.timing["d2h_bytes"] = run.io["h2d"], run.io["d2h"]
        return RunResult(output=run.output, metrics=finalize(run.trace, target.spec, draft.spec), trace=run.trace,
                         wall=run.timing)
    if use_graphs:
        run = _session_run(draft, target, prompt, config, trace_alive)
    else:
        run = DeviceRun(draft, target, prompt, config, trace_alive=trace_alive)
    t0 = time.perf_counter()
    if use_graphs:
        run.prefill()
        if run.graphs is None:
            run.capture()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        run.run_graphs()
        ev1.record()
        ev1.synchronize()
        run.timing["decode_ms"] = ev0.elapsed_time(ev1)
        run.timing["gpu_launches"] = (run.replays[0] * run.launches_per_graph[0] +
                                      run.replays[1] * run.launches_per_graph[1])
        run.timing["draft_steps"], run.timing["target_steps"] = run.replays
    else:
        run.run_stepwise()
    run.timing["wall_s"] = time.perf_counter() - t0
    run.timing["h2d_bytes"], run.timing["d2h_bytes"] = run.io["h2d"], run.io["d2h"]
    return RunResult(output=run.output, metrics=finalize(run.trace, target.spec, draft.spec), trace=run.trace,
                     wall=run.timing)


def run_speculative_batch(draft, target, prompts: Sequence[Sequence[TokenId]], config: EngineConfig,
                          ) -> tuple[list[RunResult], dict]:
    """Several requests decoded at once on one GPU (BASELINE configs[4]).

    Every request gets its own candidate tree, engine state and model
    runtimes (KV caches, activation buffers; the weights are shared) and its
    own CUDA stream; the host interleaves the requests' serial_sim cycles
    (DeviceRun.graph_cycles) so the GPU overlaps one request's
    latency-bound draft kernels with another's.  Each request follows the
    reference schedule exactly: its tokens and trace equal a single
    run_speculative of the same prompt.  Returns (results, timing) with
    timing["decode_ms"] the wall time of the interleaved decode (all
    requests) and timing["tokens"] the tokens emitted by all of them."""
    kinds = {getattr(draft, "engine_kind", "host"), getattr(target, "engine_kind", "host")}
    if kinds != {"llama"}:
        raise ConfigError("run_speculative_batch needs a transformer draft/target pair")
    if getattr(target, "tp", None) is not None:
        raise ConfigError("run_speculative_batch does not take a tensor-parallel target")
    if not config.correction_enabled or config.mode != "serial_sim":
        raise ConfigError("run_speculative_batch runs the serial_sim schedule with correction enabled")
    _validate_run_config(draft, target, config)
    runs, streams, gens = [], [], []
    for p in prompts:
        run = DeviceRun(draft, target, p, config, trace_alive=False, private_runtimes=True)
        run.prefill()
        run.capture()
        runs.append(run)
        streams.append(torch.cuda.Stream())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pending = []
    for run, st in zip(runs, streams):
        with torch.cuda.stream(st):
            g = run.graph_cycles()
            pending.append((g, next(g), st))
    while pending:
        nxt = []
        for g, ev, st in pending:
            if not ev.query():
                nxt.append((g, ev, st))
                continue
            with torch.cuda.stream(st):
                try:
                    nxt.append((g, next(g), st))
                except StopIteration:
                    pass
        pending = nxt
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - t0) * 1e3
    results = []
    for run in runs:
        run.timing.update(draft_steps=run.replays[0], target_steps=run.replays[1])
        results.append(RunResult(output=run.output, metrics=finalize(run.trace, target.spec, draft.spec),
                                 trace=run.trace, wall=run.timing))
    return results, {"decode_ms": wall_ms, "tokens": sum(len(r.output) for r in results), "requests": len(runs)}


# ====================================================================== vanilla AR
class VanillaRun:
    """Target-only autoregressive decode (engine.py:392-423) with the same
    kernels: one token per step, M = 1 rows (the 128-bit-load GEMV path)."""

    def __init__(self, target, prompt, config: EngineConfig):
        self.target_model = target
        self.cfg = config
        self.dev = require_cuda()
        self.prompt = _check_prompt(prompt, target.vocab.size)
        self.t_score = config.temperature if config.temperature > 0.0 else 1.0
        self.sampling = config.temperature > 0.0
        C0 = len(self.prompt)
        self.max_ctx = C0 + config.max_new_tokens + 8
        self.cache_capacity = 64
        # a never-expanded cache: every query misses, so each step is a miss step
        self.cache = TreeCache(self.prompt[-1], CacheConfig(1, 1, 1), eos_token=target.eos_token, capacity=64)
        order = _order_of(target)
        self.dev_d = self.dev_t = self.dev
        self.trt = _RowsAndTail(1, 1, order, self.dev)
        self.committed = torch.zeros(self.max_ctx + 8, dtype=torch.int32, device=self.dev)
        self.committed[:C0] = torch.tensor(self.prompt, dtype=torch.int32)
        rng = np.random.default_rng(config.seed)
        n_uni = config.max_new_tokens + 8 if self.sampling else 1
        self.uni = torch.from_numpy(rng.random(n_uni)).to(self.dev)
        st = EngineState()
        st.C = C0
        st.max_new = config.max_new_tokens
        st.eos = -1 if target.eos_token is None else int(target.eos_token)
        st.order = order
        st.sampling = int(self.sampling)
        st.base_len = C0
        self.E = torch.frombuffer(bytearray(bytes(st)), dtype=torch.int32).to(self.dev)
        self.E_ptr = ptr(self.E)
        self.q_tok_ptr = ctypes.c_void_p(self.cache._qbufs[1])
        self.ta = _adapter(target, "target", self, 1)
        self.graph = None

    def step(self):
        L_ = lib()
        s = stream_ptr()
        raise_for_status(L_.card_target_rows(self.E_ptr, self.cache.handle, ptr(self.committed),
                                             ptr(self.trt.rows.block), 1, 1, ptr(self.trt.tail), self.trt.order,
                                             _pt(self.ta), s),
                         "target_rows")
        self.ta.target(self)
        raise_for_status(L_.card_commit(self.E_ptr, ptr(self.committed), s), "commit")

    def prefill(self):
        self.ta.prefill(self, self.prompt[:-1])

    def capture(self):
        from . import _lib

        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            c0 = _lib.launch_count[0]
            with torch.cuda.graph(g, stream=s):
                self.step()
            self.launches_per_step = _lib.launch_count[0] - c0
        torch.cuda.current_stream().wait_stream(s)
        self.graph = g

    def decode(self, use_graph: bool = True):
        n = self.cfg.max_new_tokens
        for _ in range(n):
            if use_graph:
                self.graph.replay()
            else:
                self.step()

    def output(self) -> list[int]:
        host = self.E.cpu().numpy().tobytes()
        st = EngineState.from_buffer_copy(host)
        C0 = len(self.prompt)
        return self.committed[C0:st.C].cpu().tolist()


def run_vanilla(target, prompt: Sequence[TokenId], config: EngineConfig, *, use_graph: bool | None = None) -> RunResult:
    """engine.py:392-423 on the device."""
    if getattr(target, "engine_kind", "host") == "host":
        from .hostrun import run_vanilla_host

        return run_vanilla_host(target, prompt, config)
    run = VanillaRun(target, prompt, config)
    if use_graph is None:
        use_graph = getattr(target, "engine_kind", "") == "llama" and getattr(target, "tp", None) is None
    t0 = time.perf_counter()
    run.prefill()
    if use_graph:
        run.capture()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    run.decode(use_graph)
    ev1.record()
    ev1.synchronize()
    out = run.output()
    t_lat = target.spec.forward_latency
    trace = [StepTrace(i, (i + 1) * t_lat, False, 0, 0, 1, 0, "miss_step") for i in range(len(out))]
    wall = {"decode_ms": ev0.elapsed_time(ev1), "wall_s": time.perf_counter() - t0}
    if use_graph:
        wall["gpu_launches"] = run.cfg.max_new_tokens * run.launches_per_step
    return RunResult(output=out, metrics=finalize(trace, target.spec), trace=trace, wall=wall)


def forward_context_logits(model, context: list[int]) -> torch.Tensor:
    """Reference-API helper: logits of the last position of a full context
    (prefill-style; reuses the model's runtime KV, not reentrant)."""
    from .llama import RowBlock

    rt = model.runtime(max(len(context) + 8, 64), 0, {PREFILL_CHUNK})
    rows = RowBlock(PREFILL_CHUNK, 1, rt.dev)
    for s in range(0, len(context), PREFILL_CHUNK):
        chunk = context[s:s + PREFILL_CHUNK]
        rows.set_chain(chunk, s)
        rt.forward(rows, PREFILL_CHUNK)
    torch.cuda.synchronize()
    return rt.logits[0].clone()
