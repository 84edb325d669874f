"""Batched decode of several requests on one GPU (BASELINE configs[4],
SURVEY.md §8 f2).

The reference decodes one request at a time (engine.py:275-287; batching
across requests is a non-goal of SPEC.md:367-368).  Here B requests share
every weight stream: each draft step is ONE forward over the B requests'
frontier rows, each target step ONE verify forward over their candidate
chains.  Per request everything else stays separate and follows the
reference schedule of engine.py:290-317 (serial_sim, correction on):

* its own candidate tree (device arena + hash, cache.py), engine state,
  committed tokens, prefix KV pages and tree-KV slots, and uniforms
  (request i: default_rng(seed + i));
* its own region of the combined row blocks: ``rows_d = K + CATCH_UP``
  draft rows (frontier + catch-up), ``K`` draft outputs and
  ``query_depth + 1`` verify rows, padded when shorter
  (card_draft_rows_at / card_target_rows_at).  Catch-up rows are the
  committed tokens without draft KV: the correction token and at most one
  accepted frontier node (the accepted chain's other KV is promoted from
  tree slots, card_draft_promote), so CATCH_UP = 4 leaves margin; a request
  that overflows its region stops with a ProtocolError;
* per cycle its own number of draft expansions, min(ratio, max_depth -
  depth) (engine.py:303-310): a request whose budget or frontier runs out
  stops expanding while the others go on.

Attention reads each region's prefix through the request's page table
(card_attention_batch).  The per-request control kernels (row builders,
expand, query, verify, commit, correct, KV promotion / compaction) run on
parallel branches of the captured graphs.

``K`` is per request: a batch shares the lm_head/top-k rows of one forward,
so callers scale K down with B (``batch_config``).
A forward holds at most MAX_ROWS rows (the tcgen05 GEMM's TMEM tile);
``run_speculative_batched`` splits larger batches into sub-batches whose
cycles interleave on separate streams.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import replace
from typing import Sequence

import numpy as np
import torch

from ._device import ptr, require_cuda, stream_ptr
from ._lib import EngineState, lib
from .cache import CacheConfig, TreeCache
from .engine import (EngineConfig, RunResult, StepTrace, _check_pair, _check_prompt, _validate_run_config,
                     PREFILL_CHUNK)
from .errors import ConfigError, ProtocolError, raise_for_status
from .metrics import finalize

_SPARE0 = EngineState.spare.offset // 4   # per-cycle draft budget (card_draft_rows_at)
CATCH_UP = 4      # draft catch-up rows per request region
MAX_ROWS = 256    # rows of one forward (tc_gemm: Mpad <= 256)


def max_batch(config: EngineConfig) -> int:
    """Requests one BatchRun can hold (draft and verify regions <= MAX_ROWS)."""
    return max(1, min(MAX_ROWS // (config.K + CATCH_UP), MAX_ROWS // (config.query_depth + 1)))


def batch_config(config: EngineConfig, n_requests: int) -> EngineConfig:
    """Per-request config of a batch: the frontier budget K is shared by the
    batch (K // B per request, at least 1)."""
    return replace(config, K=max(1, config.K // max(1, n_requests)))


class BatchRun:
    """B requests decoded with shared forwards (see module docstring)."""

    BRANCHES = 8   # parallel graph branches for the per-request control kernels

    def __init__(self, draft, target, prompts: Sequence[Sequence[int]], config: EngineConfig):
        _check_pair(draft, target)
        for m in (draft, target):
            if getattr(m, "engine_kind", "") != "llama" or m.dtype != "bf16" or getattr(m, "tp", None) is not None:
                raise ConfigError("batched decode runs bf16 transformer pairs (no tensor-parallel target)")
        if not config.correction_enabled or config.mode != "serial_sim":
            raise ConfigError("batched decode runs the serial_sim schedule with correction enabled")
        _validate_run_config(draft, target, config)
        if not prompts:
            raise ConfigError("no prompts")
        self.dev = require_cuda()
        self.draft_model, self.target_model = draft, target
        self.cfg = cfg = config
        self.prompts = [_check_prompt(p, target.vocab.size) for p in prompts]
        B = self.B = len(self.prompts)
        self.sampling = cfg.temperature > 0.0
        self.t_score = cfg.temperature if self.sampling else 1.0
        self.eos = target.eos_token
        self.max_ctx = max(len(p) for p in self.prompts) + cfg.max_new_tokens + cfg.max_depth + 8
        self.cap = 6 * cfg.K * (cfg.max_depth + 1) + 256
        self.K = cfg.K
        self.k = cfg.k
        self.rd = cfg.K + CATCH_UP                 # draft rows per request (frontier + catch-up)
        self.rt_rows = cfg.query_depth + 1        # verify rows per request
        self.Md, self.Mt = B * self.rd, B * self.rt_rows
        if max(self.Md, self.Mt) > MAX_ROWS:
            raise ConfigError(f"{B} requests need {self.Md} draft / {self.Mt} verify rows per forward "
                              f"(at most {MAX_ROWS}); use run_speculative_batched, which splits the batch")
        self.XM = cfg.max_depth + 1
        order = max(1, draft.bias.order, target.bias.order)
        self.order = order
        from .llama import BatchPages, DeviceLlama, RowBlock

        dev = self.dev
        self.rt_d = DeviceLlama(draft.shard_cfg, draft.packed, max_ctx=self.max_ctx, tree_slots=B * self.cap + 1,
                                row_budgets=sorted({self.Md, PREFILL_CHUNK}), pool_requests=B,
                                extra_max=max(32, self.XM), persistent=getattr(draft, "persistent", True))
        self.rt_t = DeviceLlama(target.shard_cfg, target.packed, max_ctx=self.max_ctx, tree_slots=1,
                                row_budgets=sorted({self.Mt, PREFILL_CHUNK}), pool_requests=B,
                                persistent=getattr(target, "persistent", True))
        for rt in (self.rt_d, self.rt_t):
            if not rt.fused:
                raise ConfigError("batched decode needs the fused bf16 path")
        self.dead_d = self.rt_d.tree_base + B * self.cap
        self.dead_t = self.rt_t.tree_base
        # per-request prefix pages; the tables stacked for the batched attention
        self.pages_d = [self.rt_d.page_table(dev) for _ in range(B)]
        self.pages_t = [self.rt_t.page_table(dev) for _ in range(B)]
        self.pt_d = torch.stack([p.dev for p in self.pages_d]).contiguous()
        self.pt_t = torch.stack([p.dev for p in self.pages_t]).contiguous()
        self.bp_d = BatchPages(self.pt_d, self.pt_d.shape[1], self.rd)
        self.bp_t = BatchPages(self.pt_t, self.pt_t.shape[1], self.rt_rows)
        # trees, states, committed tokens, uniforms
        self.caches = [TreeCache(p[-1], CacheConfig(cfg.K, cfg.k, cfg.max_depth), eos_token=self.eos,
                                 capacity=self.cap) for p in self.prompts]
        rng_n = (cfg.max_new_tokens + 2) * (cfg.query_depth + 2) + 16 if self.sampling else 1
        # request i draws from default_rng(seed + i) (engine.py:162 per request):
        # request 0 of a batch samples exactly as run_speculative with the config
        self.uni = torch.from_numpy(np.stack([np.random.default_rng(cfg.seed + i).random(rng_n)
                                              for i in range(B)])).to(dev)
        states = []
        for p in self.prompts:
            st = EngineState()
            st.C = len(p)
            st.Pd = 0
            st.max_new = cfg.max_new_tokens
            st.eos = -1 if self.eos is None else int(self.eos)
            st.order = order
            st.sampling = int(self.sampling)
            st.base_len = len(p)
            st.n_uni = rng_n
            states.append(bytes(st))
        self.E = torch.frombuffer(bytearray(b"".join(states)), dtype=torch.int32).view(B, -1).to(dev)
        self._E0 = self.E.clone()   # initial states, for rebind()
        self.nE = self.E.shape[1]
        self.committed = torch.zeros((B, self.max_ctx + 8), dtype=torch.int32, device=dev)
        for i, p in enumerate(self.prompts):
            self.committed[i, :len(p)] = torch.tensor(p, dtype=torch.int32)
        self.io = {"h2d": sum(4 * len(p) for p in self.prompts) + self.uni.numel() * 8 + self.E.numel() * 4,
                   "d2h": 0}
        # combined row blocks (header = every region) and context tails
        self.rows_d = RowBlock(self.Md, self.XM, dev)
        self.rows_t = RowBlock(self.Mt, 1, dev)
        self.rows_d.block[0], self.rows_d.block[1] = self.Md, B * self.K
        self.rows_t.block[0], self.rows_t.block[1] = self.Mt, self.Mt
        self.tail_d = torch.full((self.Md, order), -1, dtype=torch.int32, device=dev)
        self.tail_t = torch.full((self.Mt, order), -1, dtype=torch.int32, device=dev)
        # draft lm_head outputs, target readers
        k = cfg.k
        self.tok = torch.zeros((self.Md, k), dtype=torch.int32, device=dev)
        self.logp = torch.zeros((self.Md, k), dtype=torch.float64, device=dev)
        self.cnt = torch.zeros(self.Md, dtype=torch.int32, device=dev)
        self.amax = torch.zeros(self.Mt, dtype=torch.int32, device=dev)
        self.lm_work_d = torch.zeros(lib().card_lmhead_work_floats(self.Md, k), dtype=torch.float32, device=dev)
        self.lm_work_t = torch.zeros(lib().card_lmhead_work_floats(self.Mt, 1), dtype=torch.float32, device=dev)
        self.probs = torch.zeros((self.Mt, target.vocab.size), dtype=torch.float64, device=dev) \
            if self.sampling else None
        # The lm_head reads its input rows as one contiguous block, but the
        # draft's output rows are spread over the requests' regions: they are
        # gathered (card_gather_rows) into a staging block the batch's own
        # lm_head linear reads.
        from .llama import EPI_STORE_F32, EPI_TOPK, TOPK_REC, _Linear

        Hd = draft.shard_cfg.hidden
        self.stage_rows = ((self.Md + 15) // 16) * 16
        self.stage_xb = torch.zeros((self.stage_rows, Hd), dtype=torch.bfloat16, device=dev)
        self.stage_ssq = torch.zeros((Hd // 16, self.stage_rows), dtype=torch.float32, device=dev)
        W = self.rt_d.lm_head
        if draft.fused_topk and k <= 4:
            n_tiles = W.shape[0] if W.dim() == 4 else W.shape[0] // 128
            work = torch.zeros(self.Md * n_tiles * TOPK_REC, dtype=torch.float32, device=dev)
            self.head = _Linear(W, self.stage_xb, self.Md, EPI_TOPK, work, 0)
            self.head.work, self.head.n_tiles = work, n_tiles
        else:
            self.head = None
            self.lm_logits = _Linear(W, self.stage_xb, self.Md, EPI_STORE_F32, self.rt_d.logits,
                                     draft.vocab.size)
        lin = self.head if self.head is not None else self.lm_logits
        lin.fuse_norm(self.stage_ssq, Hd // 16, self.stage_rows, draft.shard_cfg.rms_eps, Hd, None)
        # draft KV compaction scratch, one per request (compactions run in parallel)
        nL = draft.shard_cfg.n_layers
        row_bytes = self.rt_d.kv_row_elems() * self.rt_d.kv_esize()
        self.scratch = []
        for _ in range(B):
            sk = torch.zeros(self.cap * nL * row_bytes // 2, dtype=torch.int16, device=dev)
            sv = torch.zeros_like(sk)
            self.scratch.append((sk, sv, torch.tensor([sk.data_ptr(), sv.data_ptr()], dtype=torch.int64, device=dev)))
        self._host = torch.empty((B, self.nE), dtype=torch.int32, pin_memory=True)
        self._budget = torch.empty(B, dtype=torch.int32, pin_memory=True)
        self.branches = [torch.cuda.Stream() for _ in range(min(B, self.BRANCHES))]
        self.outputs: list[list[int]] = [[] for _ in range(B)]
        self.traces: list[list[StepTrace]] = [[] for _ in range(B)]
        self.graphs = None
        self.timing: dict = {}

    def rebind(self, prompts: Sequence[Sequence[int]]):
        """A new batch of prompts (same count and lengths) on this run's
        buffers and captured graphs: every buffer a step could read goes back
        to its constructor contents (trees cleared, states, committed tokens,
        tails, reader outputs); call prefill() next."""
        prompts = [_check_prompt(p, self.target_model.vocab.size) for p in prompts]
        if [len(p) for p in prompts] != [len(p) for p in self.prompts]:
            raise ConfigError("rebind needs prompts of the run's lengths")
        self.prompts = prompts
        for c, p in zip(self.caches, prompts):
            c.clear(p[-1])
        self.E.copy_(self._E0)
        self.committed.zero_()
        for i, p in enumerate(prompts):
            self.committed[i, :len(p)] = torch.tensor(p, dtype=torch.int32)
        self.tail_d.fill_(-1)
        self.tail_t.fill_(-1)
        for t in (self.tok, self.logp, self.cnt, self.amax, self.lm_work_d, self.lm_work_t, self.probs):
            if t is not None:
                t.zero_()
        self.io = {"h2d": sum(4 * len(p) for p in prompts) + self.E.numel() * 4, "d2h": 0}
        self.outputs = [[] for _ in range(self.B)]
        self.traces = [[] for _ in range(self.B)]
        if self.graphs is not None:
            self.replays = [0, 0]

    # ------------------------------------------------------------ helpers
    def _Ep(self, i: int, field: str | None = None) -> ctypes.c_void_p:
        off = 0 if field is None else getattr(EngineState, field).offset
        return ctypes.c_void_p(self.E.data_ptr() + i * self.nE * 4 + off)

    def _bias_args(self, model, tail: torch.Tensor) -> tuple:
        b = model.bias
        if b.sharpness == 0.0:
            return (None, 0, 0, 0, 0, 0.0, 0.0)
        M64 = (1 << 64) - 1
        return (ctypes.c_void_p(tail.data_ptr() + 4 * (self.order - b.order)), b.order, self.order, b.seed & M64,
                b.mix_seed & M64, float(b.mix_weight), float(b.sharpness))

    def _fan_out(self, fn):
        """fn(i) for every request on parallel branches of the current stream
        (graph capture records them as concurrent nodes), joined after."""
        main = torch.cuda.current_stream()
        for st in self.branches:
            st.wait_stream(main)
        for i in range(self.B):
            with torch.cuda.stream(self.branches[i % len(self.branches)]):
                fn(i)
        for st in self.branches:
            main.wait_stream(st)

    # ------------------------------------------------------------ prefill
    def prefill(self):
        """Each request's prompt[:-1] into its prefix pages of both models."""
        from .llama import RowBlock

        rows = RowBlock(PREFILL_CHUNK, 1, self.dev)
        for i, p in enumerate(self.prompts):
            body = p[:-1]
            for rt, pages in ((self.rt_d, self.pages_d[i]), (self.rt_t, self.pages_t[i])):
                for s in range(0, len(body), PREFILL_CHUNK):
                    self.io["h2d"] += rows.set_chain(body[s:s + PREFILL_CHUNK], s, pages=pages)
                    rt.forward(rows, PREFILL_CHUNK, pages=pages)
            self.E[i, EngineState.Pd.offset // 4] = len(body)
        self.io["h2d"] += 4 * self.B

    # ------------------------------------------------------------ steps
    def launch_draft_step(self):
        L_ = lib()
        cfg = self.cfg
        K, rd, k = self.K, self.rd, self.k

        def rows(i):
            c = self.caches[i]
            raise_for_status(L_.card_draft_rows_at(
                self._Ep(i), c.handle, ptr(self.committed[i]), ptr(self.rows_d.block), self.Md, self.XM, i * rd, rd,
                i * K, K, self.dead_d, self.rt_d.tree_base + i * self.cap, ptr(self.tail_d), self.order,
                ptr(self.pt_d[i]), stream_ptr()), "draft_rows_at")

        self._fan_out(rows)
        bias = self._bias_args(self.draft_model, self.tail_d)
        n_out = self.rows_d.n_out
        rt = self.rt_d
        rt.forward(self.rows_d, self.Md, batch=self.bp_d, head=False)
        raise_for_status(L_.card_gather_rows(ptr(self.rows_d.out_rows), ptr(n_out), self.Md,
                                             self.draft_model.shard_cfg.hidden, ptr(rt.xb), ptr(rt.ssq), rt.mpad,
                                             ptr(self.stage_xb), ptr(self.stage_ssq), self.stage_rows, stream_ptr()),
                         "gather_rows")
        if self.head is not None:
            head = self.head
            raise_for_status(L_.card_linear_fuse_kgram(head.h, *bias), "fuse_kgram")
            raise_for_status(L_.card_linear_fuse_topk(head.h, self.draft_model.vocab.size, 1.0 / self.t_score),
                             "fuse_topk")
            head.run(n_out)
            raise_for_status(L_.card_lmhead_topk_merge(ptr(head.work), ptr(n_out), self.Md, head.n_tiles, k,
                                                       self.draft_model.vocab.size, ptr(self.tok), ptr(self.logp),
                                                       ptr(self.cnt), stream_ptr()), "lmhead_topk_merge")
        else:
            self.lm_logits.run(n_out)
            raise_for_status(L_.card_topk_logits(ptr(self.rt_d.logits), ptr(n_out), self.Md,
                                                 self.draft_model.vocab.size, k, 1.0 / self.t_score, ptr(self.tok),
                                                 ptr(self.logp), ptr(self.cnt), ptr(self.lm_work_d), *bias,
                                                 stream_ptr()), "topk_logits")

        def expand(i):
            c = self.caches[i]
            raise_for_status(L_.card_cache_expand_topk(
                c.handle, ctypes.c_void_p(self.tok.data_ptr() + i * K * k * 4),
                ctypes.c_void_p(self.logp.data_ptr() + i * K * k * 8), ctypes.c_void_p(self.cnt.data_ptr() + i * K * 4),
                -1, 0, self._Ep(i, "stop"), stream_ptr()), "expand")
            raise_for_status(L_.card_record_width(self._Ep(i), c.handle, ptr(n_out), stream_ptr()), "record")

        self._fan_out(expand)

    def launch_target_step(self):
        L_ = lib()
        cfg = self.cfg
        R = self.rt_rows

        def rows(i):
            c = self.caches[i]
            raise_for_status(L_.card_cache_query(c.handle, cfg.query_depth, stream_ptr()), "query")
            raise_for_status(L_.card_target_rows_at(
                self._Ep(i), c.handle, ptr(self.committed[i]), ptr(self.rows_t.block), self.Mt, 1, i * R, R,
                self.dead_t, ptr(self.tail_t), self.order, ptr(self.pt_t[i]), stream_ptr()), "target_rows_at")

        self._fan_out(rows)
        self.rt_t.forward(self.rows_t, self.Mt, batch=self.bp_t)
        V = self.target_model.vocab.size
        bias = self._bias_args(self.target_model, self.tail_t)
        if self.sampling:
            if bias[6] != 0.0:
                raise_for_status(L_.card_logit_bias(ptr(self.rt_t.logits), ptr(self.rows_t.n_out), self.Mt, V, *bias,
                                                    stream_ptr()), "logit_bias")
            raise_for_status(L_.card_softmax64(ptr(self.rt_t.logits), ptr(self.rows_t.n_out), self.Mt, V,
                                               1.0 / self.t_score, ptr(self.probs), stream_ptr()), "softmax64")
        else:
            raise_for_status(L_.card_argmax_logits(ptr(self.rt_t.logits), ptr(self.rows_t.n_out), self.Mt, V,
                                                   ptr(self.amax), ptr(self.lm_work_t), *bias, stream_ptr()), "argmax")
        nL = self.draft_model.shard_cfg.n_layers
        rt_d = self.rt_d

        def verify_commit_correct(i):
            c = self.caches[i]
            E = self._Ep(i)
            q_tok = ctypes.c_void_p(c._qbufs[1])
            if self.sampling:
                raise_for_status(L_.card_verify_probs(E, q_tok, ctypes.c_void_p(self.probs.data_ptr() + i * R * V * 8),
                                                      V, None, ptr(self.uni[i]), stream_ptr()), "verify_probs")
            else:
                raise_for_status(L_.card_verify_argmax(E, q_tok, ctypes.c_void_p(self.amax.data_ptr() + i * R * 4),
                                                       stream_ptr()), "verify_argmax")
            raise_for_status(L_.card_commit(E, ptr(self.committed[i]), stream_ptr()), "commit")
            raise_for_status(L_.card_cache_correct(c.handle, self._Ep(i, "acc"), self._Ep(i, "n_acc"),
                                                   self._Ep(i, "corr"), self._Ep(i, "done"), stream_ptr()), "correct")
            tb = rt_d.tree_base + i * self.cap
            raise_for_status(L_.card_draft_promote(E, c.handle, ptr(rt_d.k_ptrs), ptr(rt_d.v_ptrs), nL,
                                                   rt_d.kv_row_elems(), rt_d.kv_esize(), tb, self.cfg.max_depth + 2,
                                                   ptr(self.pt_d[i]), stream_ptr()), "draft_promote")
            raise_for_status(L_.card_kv_compact(E, c.handle, ptr(rt_d.k_ptrs), ptr(rt_d.v_ptrs), nL,
                                                rt_d.kv_row_elems(), rt_d.kv_esize(), tb, ptr(self.scratch[i][2]),
                                                self.cap, stream_ptr()), "kv_compact")
            raise_for_status(L_.card_cycle_end(E, c.handle, stream_ptr()), "cycle_end")

        self._fan_out(verify_commit_correct)
        self._host.copy_(self.E, non_blocking=True)

    # ------------------------------------------------------------ driver
    def capture(self):
        from . import _lib

        g_d, g_t = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            c0 = _lib.launch_count[0]
            with torch.cuda.graph(g_d, stream=s):
                self.launch_draft_step()
            c1 = _lib.launch_count[0]
            with torch.cuda.graph(g_t, stream=s):
                self.launch_target_step()
            c2 = _lib.launch_count[0]
        torch.cuda.current_stream().wait_stream(s)
        self.graphs = (g_d, g_t)
        self.launches_per_graph = (c1 - c0, c2 - c1)
        self.replays = [0, 0]

    def _set_budgets(self, budgets: list[int]):
        self._budget.copy_(torch.tensor(budgets, dtype=torch.int32))
        self.E[:, _SPARE0].copy_(self._budget, non_blocking=True)
        self.io["h2d"] += 4 * self.B

    @staticmethod
    def _event():
        ev = torch.cuda.Event()
        ev.record()
        return ev

    def _read(self) -> list[EngineState]:
        """The states copied at the end of the last cycle (its event completed)."""
        self.io["d2h"] += self.E.numel() * 4
        raw = self._host.numpy()
        out = [EngineState.from_buffer_copy(raw[i].tobytes()) for i in range(self.B)]
        for i, E in enumerate(out):
            if E.done < 0:
                raise ProtocolError(f"request {i}: draft rows overflow the batch row region ({self.rd} rows)")
        return out

    def run(self):
        """The serial_sim schedule of every request (engine.py:290-317), the
        requests' steps sharing each forward; one host round trip per cycle."""
        for ev in self.cycles():
            ev.synchronize()

    def cycles(self):
        """run() as a generator: each cycle launches its graphs on the current
        stream, records an event and yields it; resume once it completed."""
        cfg = self.cfg
        d_lat = self.draft_model.spec.forward_latency
        t_lat = self.target_model.spec.forward_latency
        g_d, g_t = self.graphs
        B = self.B
        clock = [0.0] * B
        depth = [0] * B
        self._set_budgets([cfg.query_depth] * B)
        for _ in range(cfg.query_depth):   # warm-up (engine.py:295-301)
            g_d.replay()
            self.replays[0] += 1
        self._host.copy_(self.E, non_blocking=True)
        yield self._event()
        for i, E in enumerate(self._read()):
            for w in list(E.widths)[:min(E.n_widths, 64)]:
                if w == 0:
                    break
                depth[i] += 1
                clock[i] += d_lat
                self.traces[i].append(StepTrace(len(self.traces[i]), clock[i], False, int(w), 0, 0, -1, "draft_expand"))
        self.E[:, EngineState.n_widths.offset // 4] = 0
        self.E[:, EngineState.stop.offset // 4] = 0
        live = [True] * B
        while any(live):
            budgets = [min(cfg.ratio, max(0, cfg.max_depth - depth[i])) if live[i] else 0 for i in range(B)]
            self._set_budgets(budgets)
            for _ in range(max(budgets)):
                g_d.replay()
            g_t.replay()
            self.replays[0] += max(budgets)
            self.replays[1] += 1
            yield self._event()
            for i, E in enumerate(self._read()):
                if not live[i]:
                    continue
                tr = self.traces[i]
                start, kk = clock[i], 0
                for w in list(E.rec_widths)[:min(E.rec_n_widths, 64)]:
                    if w == 0:
                        break
                    kk += 1
                    tr.append(StepTrace(len(tr), start + kk * d_lat, False, int(w), 0, 0, -1, "draft_expand"))
                clock[i] = start + max(kk * d_lat, t_lat)
                hit = bool(E.rec_hit)
                self.outputs[i].extend(E.committed_now[j] for j in range(E.n_commit))
                tr.append(StepTrace(len(tr), clock[i], hit, E.rec_L if hit else 0, E.rec_acc, E.rec_lnew, -1,
                                    "verify" if hit else "miss_step"))
                if E.rec_done:
                    live[i] = False
                else:
                    tr.append(StepTrace(len(tr), clock[i], hit, 0, 0, 0, -1, "correct"))
                depth[i] = E.rec_depth


_SESSIONS_PER_TARGET = 4


def _session(draft, target, prompts, config: EngineConfig, slot: int) -> BatchRun:
    """A serving session per (pair, prompt lengths, config, sub-batch slot):
    the BatchRun's buffers and captured graphs are built by the first batch
    and rebound to the next ones, as a server captures its graphs once per
    shape (engine._session_run does the same for single requests)."""
    from .engine import _model_sig

    key = (_model_sig(draft), _model_sig(target), tuple(len(p) for p in prompts),
           tuple(sorted(config.to_dict().items())), slot)
    store = target.__dict__.setdefault("_card_batch_sessions", {})
    run = store.pop(key, None)
    if run is not None and run.draft_model is draft:
        run.rebind(prompts)
    else:
        run = BatchRun(draft, target, prompts, config)
    store[key] = run
    while len(store) > _SESSIONS_PER_TARGET:
        store.pop(next(iter(store)))
    return run


def run_speculative_batched(draft, target, prompts: Sequence[Sequence[int]], config: EngineConfig,
                            ) -> tuple[list[RunResult], dict]:
    """Decode every prompt with shared draft / verify forwards (BatchRun).
    ``config`` is per request (see batch_config).  Batches larger than
    max_batch(config) run as sub-batches whose cycles interleave on their
    own streams.  Returns (results, timing): timing["decode_ms"] is the
    device time of the whole decode, timing["tokens"] the tokens all
    requests emitted."""
    per = max_batch(config)
    groups = [list(prompts[j:j + per]) for j in range(0, len(prompts), per)]
    runs = [_session(draft, target, g, config, j) for j, g in enumerate(groups)]
    streams = [torch.cuda.Stream() for _ in runs]
    for run in runs:
        run.prefill()
        if run.graphs is None:
            run.capture()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    pending = []
    for run, st in zip(runs, streams):
        st.wait_event(ev0)
        with torch.cuda.stream(st):
            gen = run.cycles()
            pending.append((gen, next(gen), st))
    while pending:
        nxt = []
        for gen, ev, st in pending:
            if not ev.query():
                nxt.append((gen, ev, st))
                continue
            with torch.cuda.stream(st):
                try:
                    nxt.append((gen, next(gen), st))
                except StopIteration:
                    pass
        pending = nxt
    for st in streams:
        torch.cuda.current_stream().wait_stream(st)
    ev1.record()
    ev1.synchronize()
    wall = time.perf_counter() - t0
    lpg = runs[0].launches_per_graph
    timing = {"decode_ms": ev0.elapsed_time(ev1), "wall_s": wall, "requests": len(prompts), "sub_batches": len(runs),
              "tokens": sum(len(o) for r in runs for o in r.outputs),
              "draft_steps": sum(r.replays[0] for r in runs), "target_steps": sum(r.replays[1] for r in runs),
              "gpu_launches": sum(r.replays[0] * r.launches_per_graph[0] + r.replays[1] * r.launches_per_graph[1]
                                  for r in runs),
              "launches_per_graph": lpg, "h2d_bytes": sum(r.io["h2d"] for r in runs),
              "d2h_bytes": sum(r.io["d2h"] for r in runs), "K_per_request": config.K}
    results = [RunResult(output=o, metrics=finalize(t, target.spec, draft.spec), trace=t, wall=timing)
               for r in runs for o, t in zip(r.outputs, r.traces)]
    return results, timing
