"""Llama-architecture draft/target models on the device.

The reference's model plug-in is the ``ToyModel`` duck type
(/root/reference/pkg/src/specache/lm.py:109-196): ``next_distribution``
over a full context and ``batch_tree_forward`` over the newest tree layer.
Here a model is a KV-cached forward over *rows* built on the device by the
engine (csrc/card_engine.cu): causal chain rows (prefill, target verify,
draft catch-up) and tree rows (one per frontier node, attending to the
committed prefix plus its own ancestors).  Every op is a kernel of
libcard_b200.so; the weights stream through the tcgen05/TMA GEMM.

Weight layout in HBM (bf16 production / fp32 parity):
  embed [V,H]; per layer wqkv [(nh+2nkv)*hd, H] (+ fp32 bias for Qwen2),
  wo [H, nh*hd], wgu [2F, H] interleaved per 32-row block (16 gate rows then
  the 16 matching up rows), wd [H, F], fp32 norms; lm_head [V,H] (tied for
  Llama-3.2-1B / Qwen2.5-0.5B).  KV cache per layer: K,V [slots, nkv, hd]
  with slots = prefix positions (rounded to 64) + draft tree slots.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field, asdict

import numpy as np
import torch

from ._device import ptr, require_cuda, stream_ptr
from ._lib import lib
from .errors import ConfigError, raise_for_status

EPI_STORE_F32, EPI_RESID_F32, EPI_STORE_BF16, EPI_SWIGLU_BF16, EPI_QKV_ROPE, EPI_TOPK = 0, 1, 2, 3, 4, 5
TOPK_REC = 10   # floats per (row, vocab tile) record of an EPI_TOPK lm_head (csrc/card_llm.h kTopkRec)


@dataclass
class LlamaConfig:
    vocab_size: int
    hidden: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    rope_theta: float = 500000.0
    rms_eps: float = 1e-5
    tie_embeddings: bool = False
    qkv_bias: bool = False
    rope_scaling: dict | None = None
    init_std: float = 0.02

    def __post_init__(self):
        if self.n_heads % self.n_kv_heads:
            raise ConfigError("n_heads must be a multiple of n_kv_heads")
        if self.head_dim % 2:
            raise ConfigError("head_dim must be even")
        if self.ffn % 64:
            raise ConfigError("ffn must be a multiple of 64 (gate/up tile interleave)")

    @property
    def qkv_dim(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    def layer_params(self) -> int:
        H, F = self.hidden, self.ffn
        return H * self.qkv_dim + (self.qkv_dim if self.qkv_bias else 0) + self.n_heads * self.head_dim * H \
            + 3 * H * F + 2 * H

    def stream_params(self) -> int:
        """Parameters streamed per forward: layers + final norm + lm_head."""
        return self.n_layers * self.layer_params() + self.hidden + self.vocab_size * self.hidden

    def total_params(self) -> int:
        emb = self.vocab_size * self.hidden
        return self.stream_params() + (0 if self.tie_embeddings else emb)

    def to_dict(self) -> dict:
        return asdict(self)


_LLAMA3_SCALING_1B = dict(factor=32.0, low_freq_factor=1.0, high_freq_factor=4.0,
                          original_max_position_embeddings=8192)
_LLAMA3_SCALING_8B = dict(factor=8.0, low_freq_factor=1.0, high_freq_factor=4.0,
                          original_max_position_embeddings=8192)

PRESETS = {
    # BASELINE.json configs[1]
    "llama-3.2-1b": LlamaConfig(128256, 2048, 16, 32, 8, 64, 8192, 500000.0, 1e-5, True, False, _LLAMA3_SCALING_1B),
    "llama-3.1-8b": LlamaConfig(128256, 4096, 32, 32, 8, 128, 14336, 500000.0, 1e-5, False, False, _LLAMA3_SCALING_8B),
    # BASELINE.json configs[3] (tensor-parallel target, tp.py)
    "llama-3.1-70b": LlamaConfig(128256, 8192, 80, 64, 8, 128, 28672, 500000.0, 1e-5, False, False, _LLAMA3_SCALING_8B),
    # BASELINE.json configs[2].  The two checkpoints pad their embedding tables
    # differently (151936 vs 152064 rows) over one 151665-token tokenizer; the
    # engine needs one vocabulary (engine.py:127-136), so the draft is padded
    # to the target's 152064 rows (padding rows are never real tokens).
    "qwen2.5-0.5b": LlamaConfig(152064, 896, 24, 14, 2, 64, 4864, 1000000.0, 1e-6, True, True, None),
    "qwen2.5-7b": LlamaConfig(152064, 3584, 28, 28, 4, 128, 18944, 1000000.0, 1e-6, False, True, None),
    # BASELINE.json configs[0]: the CPU-runnable tiny pair (FFN rounded to 704)
    "tiny-target": LlamaConfig(64, 256, 4, 4, 2, 64, 704, 10000.0, 1e-5, False, False, None),
    "tiny-draft": LlamaConfig(64, 128, 2, 4, 2, 32, 384, 10000.0, 1e-5, False, False, None),
    # bf16-kernel test sizes (multiples of the 128x64 weight tile)
    "small-target": LlamaConfig(512, 512, 4, 8, 4, 64, 1536, 10000.0, 1e-5, False, False, None),
    "small-draft": LlamaConfig(512, 256, 2, 4, 2, 64, 768, 10000.0, 1e-5, True, False, None),
}


def rope_tables(cfg: LlamaConfig, max_pos: int) -> tuple[torch.Tensor, torch.Tensor]:
    """cos/sin [max_pos, hd/2] fp32, HF Llama-3 frequency scaling; computed on
    the CPU so the device and the oracle use identical tables."""
    hd = cfg.head_dim
    inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.int64).float() / hd))
    sc = cfg.rope_scaling
    if sc:
        factor, lo, hi, old = sc["factor"], sc["low_freq_factor"], sc["high_freq_factor"], \
            sc["original_max_position_embeddings"]
        low_wl, high_wl = old / lo, old / hi
        wl = 2 * math.pi / inv
        inv_l = torch.where(wl > low_wl, inv / factor, inv)
        smooth = (old / wl - lo) / (hi - lo)
        smoothed = (1 - smooth) * inv_l / factor + smooth * inv_l
        is_med = ~(wl < high_wl) * ~(wl > low_wl)
        inv = torch.where(is_med, smoothed, inv_l)
    t = torch.arange(max_pos, dtype=torch.int64).float()
    freqs = torch.outer(t, inv)
    return freqs.cos().contiguous(), freqs.sin().contiguous()


def iter_weights(cfg: LlamaConfig, seed: int, device="cpu", dtype=torch.float32):
    """(name, tensor) of the canonical random-init weights in generation
    order (one seeded generator): Normal(0, init_std), norms 1, biases 0.
    A tied lm_head is not yielded (it is the embedding)."""
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))

    def normal(*shape):
        t = torch.empty(shape, dtype=torch.float32, device=device)
        t.normal_(0.0, cfg.init_std, generator=g)
        return t.to(dtype)

    H, hd = cfg.hidden, cfg.head_dim
    yield "embed", normal(cfg.vocab_size, H)
    for i in range(cfg.n_layers):
        p = f"l{i}."
        yield p + "wq", normal(cfg.n_heads * hd, H)
        yield p + "wk", normal(cfg.n_kv_heads * hd, H)
        yield p + "wv", normal(cfg.n_kv_heads * hd, H)
        if cfg.qkv_bias:
            yield p + "bq", torch.zeros(cfg.n_heads * hd, device=device)
            yield p + "bk", torch.zeros(cfg.n_kv_heads * hd, device=device)
            yield p + "bv", torch.zeros(cfg.n_kv_heads * hd, device=device)
        yield p + "wo", normal(H, cfg.n_heads * hd)
        yield p + "wg", normal(cfg.ffn, H)
        yield p + "wu", normal(cfg.ffn, H)
        yield p + "wd", normal(H, cfg.ffn)
        yield p + "attn_norm", torch.ones(H, device=device)
        yield p + "mlp_norm", torch.ones(H, device=device)
    yield "norm", torch.ones(H, device=device)
    if not cfg.tie_embeddings:
        yield "lm_head", normal(cfg.vocab_size, H)


def init_weights(cfg: LlamaConfig, seed: int, device="cpu", dtype=torch.float32) -> dict:
    """Canonical (HF-layout) random-init weights (iter_weights).  Same seed +
    same device => identical tensors (the oracle and the device model are
    built from one call on the CPU for parity runs)."""
    w = dict(iter_weights(cfg, seed, device, dtype))
    if cfg.tie_embeddings:
        w["lm_head"] = w["embed"]
    return w


def tile_sw128(w: torch.Tensor) -> torch.Tensor:
    """Row-major bf16 [N, K] -> pre-tiled [N/128, K/64, 128, 64] blocks with the
    SWIZZLE_128B XOR applied (16-byte chunk c of row r stored at c ^ (r % 8)),
    so one contiguous 16 KB bulk copy lands exactly as a swizzled TMA tile."""
    N, K = w.shape
    t = w.view(N // 128, 128, K // 64, 64).permute(0, 2, 1, 3)          # [nt, kb, 128, 64]
    t = t.reshape(N // 128, K // 64, 128, 8, 8)                          # chunks of 8 bf16 (16 B)
    r = torch.arange(128, device=w.device).view(128, 1)
    j = torch.arange(8, device=w.device).view(1, 8)
    src = (j ^ (r % 8)).expand(128, 8)                                   # new[r, j] = old[r, j ^ (r%8)]
    idx = src.view(1, 1, 128, 8, 1).expand(N // 128, K // 64, 128, 8, 8)
    return torch.gather(t, 3, idx).reshape(N // 128, K // 64, 128, 64).contiguous()


def interleave_gate_up(wg: torch.Tensor, wu: torch.Tensor) -> torch.Tensor:
    """[2F, H]: per 32-row block, 16 gate rows then the 16 matching up rows, so
    one epilogue warp (32 TMEM lanes) holds both halves of its 16 features."""
    F, H = wg.shape
    t = torch.stack([wg.view(F // 16, 16, H), wu.view(F // 16, 16, H)], dim=1)
    return t.reshape(2 * F, H).contiguous()


def pack_weights(cfg: LlamaConfig, weights: dict, dtype: str = "bf16", device=None) -> dict:
    """Canonical weights -> the device layout (fused QKV, interleaved gate/up).

    bf16: each RMSNorm weight is folded into the columns of the linear that
    consumes the normalised activations (W' = W diag(w): attn_norm -> wqkv,
    mlp_norm -> wgu, final norm -> lm_head); the GEMM then consumes the bf16
    residual and applies the per-token rsqrt(mean x^2 + eps) in its epilogue
    (card_linear_fuse_norm).  fp32 parity weights stay unfolded."""
    if dtype not in ("bf16", "fp32"):
        raise ConfigError(f"dtype must be bf16 or fp32, got {dtype!r}")
    dev = device or require_cuda()
    wdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    to = lambda t: t.to(device=dev, dtype=wdt).contiguous()  # noqa: E731
    f32 = lambda t: t.to(device=dev, dtype=torch.float32).contiguous()  # noqa: E731
    # bf16 linear weights live pre-tiled (tile_sw128); fp32 parity weights row-major
    lin = (lambda t: tile_sw128(to(t))) if dtype == "bf16" else to  # noqa: E731
    fold = dtype == "bf16"
    col = (lambda w, g: w.float() * g.float().view(1, -1)) if fold else (lambda w, g: w)  # noqa: E731
    out = {"dtype": dtype, "embed": to(weights["embed"]), "norm": f32(weights["norm"]), "layers": [],
           "folded": fold}
    out["lm_head"] = lin(col(weights["lm_head"].to(dev), weights["norm"].to(dev)))
    for i in range(cfg.n_layers):
        p = f"l{i}."
        out["layers"].append({
            "wqkv": lin(col(torch.cat([weights[p + "wq"], weights[p + "wk"], weights[p + "wv"]], 0).to(dev),
                            weights[p + "attn_norm"].to(dev))),
            "wo": lin(weights[p + "wo"]),
            "wgu": lin(col(interleave_gate_up(weights[p + "wg"], weights[p + "wu"]).to(dev),
                           weights[p + "mlp_norm"].to(dev))),
            "wd": lin(weights[p + "wd"]),
            "attn_norm": f32(weights[p + "attn_norm"]),
            "mlp_norm": f32(weights[p + "mlp_norm"]),
            "bqkv": f32(torch.cat([weights[p + "bq"], weights[p + "bk"], weights[p + "bv"]], 0))
            if cfg.qkv_bias else None,
        })
    return out


class _Linear:
    def __init__(self, W: torch.Tensor, X: torch.Tensor, m_max: int, epi: int, out: torch.Tensor, ldo: int,
                 bias: torch.Tensor | None = None):
        """W: row-major [N, K] (bf16 or fp32) or pre-tiled bf16 [N/128, K/64, 128, 64]."""
        self.keep = (W, X, out, bias)
        self._swiglu = epi == EPI_SWIGLU_BF16
        h = ctypes.c_void_p()
        if W.dim() == 4:
            wd, N, K = 2, W.shape[0] * 128, W.shape[1] * 64
        else:
            wd, N, K = (0 if W.dtype == torch.bfloat16 else 1), W.shape[0], W.shape[1]
        self.N, self.K = N, K
        self.nbytes = N * K * W.element_size()
        rc = lib().card_linear_create(ptr(W), N, K, wd, ptr(X), m_max, epi, ptr(out), ldo, ptr(bias),
                                      ctypes.byref(h))
        raise_for_status(rc, f"card_linear_create(N={N}, K={K}, m_max={m_max})")
        self.h = h
        info = (ctypes.c_int32 * 8)()
        lib().card_linear_info(h, info)
        self.info = dict(zip(("kind", "splits", "stages", "grid", "smem", "Mpad", "tmem_cols", "items"), list(info)))

    def fuse_norm(self, ssq: torch.Tensor, parts: int, ld: int, eps: float, H: int, x_row_off=None):
        raise_for_status(lib().card_linear_fuse_norm(self.h, ptr(ssq), parts, ld, eps, H, ptr(x_row_off)),
                         "card_linear_fuse_norm")

    def fuse_resid(self, ssq: torch.Tensor, ld: int, xb: torch.Tensor):
        raise_for_status(lib().card_linear_fuse_resid(self.h, ptr(ssq), ld, ptr(xb)), "card_linear_fuse_resid")

    def fuse_rope(self, rows, cos, sin, nh, nkv, hd, q, kc, vc):
        raise_for_status(lib().card_linear_fuse_rope(self.h, ptr(rows.pos), ptr(rows.slot), ptr(cos), ptr(sin), nh, nkv,
                                                     hd, ptr(q), ptr(kc), ptr(vc)), "card_linear_fuse_rope")

    def run(self, dM: torch.Tensor):
        from . import _lib

        _lib.launch_count[0] += 2 if (self.info["kind"] != 0 and self.keep and self._swiglu) else 1
        rc = lib().card_linear_run(self.h, ptr(dM), stream_ptr())
        if rc:
            raise_for_status(rc, "card_linear_run")

    def __del__(self):
        try:
            if self.h:
                lib().card_linear_destroy(self.h)
        except Exception:
            pass


PAGE = 64   # KV slots per page


class PagePool:
    """Free list of the prefix KV pages of one runtime.  Every request
    (DeviceRun / VanillaRun) takes the pages of its context from here and
    returns them when it is dropped; its page table maps logical page i of
    its context to a physical page.  Pages come out lowest-first, so a
    fragmented pool hands a request scattered, out-of-order pages — which
    the kernels (row builders, attention, KV promotion) only ever see
    through the table."""

    def __init__(self, n_pages: int):
        self.n_pages = n_pages
        self.free = list(range(n_pages))

    def alloc(self, n: int) -> list[int]:
        if n > len(self.free):
            import gc

            gc.collect()   # runs that died in reference cycles give their pages back
        if n > len(self.free):
            raise ConfigError(f"KV page pool exhausted: {n} pages wanted, {len(self.free)} of {self.n_pages} free")
        self.free.sort()
        out, self.free = self.free[:n], self.free[n:]
        return out

    def release(self, pages) -> None:
        self.free.extend(int(p) for p in pages)


class PageTable:
    """One request's pages (host list + device int32 table); returns them to
    the pool when collected."""

    def __init__(self, pool: PagePool, n_pages: int, device):
        self.pool = pool
        self.pages = pool.alloc(n_pages)
        self.dev = torch.tensor(self.pages, dtype=torch.int32, device=device)

    def slot(self, p: int) -> int:
        return self.pages[p // PAGE] * PAGE + p % PAGE

    def __del__(self):
        try:
            self.pool.release(self.pages)
        except Exception:
            pass


class _PFwd:
    """Persistent wide forward (csrc/card_pfwd.cu): the o / gate-up / down /
    next-qkv GEMMs of a layer in one cooperative launch, weights streaming
    across the step boundaries.  Used for wide row budgets (draft tree steps)."""

    PHASES = 5   # qkv, attention, o, gate/up, down

    def __init__(self, rt: "DeviceLlama", m_max: int):
        c = rt.cfg
        n = c.n_layers
        W = (ctypes.c_void_p * (4 * n))()
        B = (ctypes.c_void_p * n)()
        KV = (ctypes.c_void_p * (2 * n))()
        for i, L in enumerate(rt.layers):
            for j, key in enumerate(("wqkv", "wo", "wgu", "wd")):
                W[4 * i + j] = ptr(L[key])
            B[i] = ptr(L["bqkv"]) if L["bqkv"] is not None else None
            KV[2 * i], KV[2 * i + 1] = ptr(rt.k_cache[i]), ptr(rt.v_cache[i])
        h = ctypes.c_void_p()
        rc = lib().card_pfwd_create(n, c.hidden, c.ffn, c.n_heads, c.n_kv_heads, c.head_dim, m_max,
                                    ctypes.cast(W, ctypes.c_void_p), ctypes.cast(B, ctypes.c_void_p),
                                    ctypes.cast(KV, ctypes.c_void_p), ptr(rt.x), ptr(rt.xb), ptr(rt.ssq), rt.mpad,
                                    ptr(rt.q), ptr(rt.o), ptr(rt.g), rt.mpad, ptr(rt.rows_placeholder),
                                    ptr(rt.rows_placeholder), ptr(rt.cos), ptr(rt.sin), c.rms_eps, ctypes.byref(h))
        raise_for_status(rc, f"card_pfwd_create(m_max={m_max})")
        self.h = h
        self.n_layers = n
        # the qkv epilogue hands the attention its Q operand as pre-swizzled
        # bf16 tiles (card_attention_tree: one bulk copy per tile)
        # (per forward, when the row block's extras fit the tcgen05 kernel:
        # use_qsw; otherwise q stays fp32 for card_attention_paged)
        G = c.n_heads // c.n_kv_heads
        self.G = G
        self.qsw = None
        self.qsw_on = False
        if c.head_dim in (64, 128) and (128 // G + 2) <= 136:
            self.qsw_tiles = (rt.mpad * G + 127) // 128
            self.qsw = torch.zeros(c.n_kv_heads * self.qsw_tiles * (c.head_dim // 64) * 16384, dtype=torch.uint8,
                                   device=rt.dev)

    def use_qsw(self, extra_max: int) -> bool:
        """Route Q through the pre-swizzled tiles for this forward's rows (the
        setting is copied into each launch, so captured graphs keep it)."""
        on = self.qsw is not None and (128 // self.G + 2) * extra_max <= 1024
        if on != self.qsw_on:
            raise_for_status(lib().card_pfwd_set_qsw(self.h, ptr(self.qsw) if on else None,
                                                     self.qsw_tiles if on else 0), "card_pfwd_set_qsw")
            self.qsw_on = on
        return on

    def bind(self, rows: "RowBlock"):
        raise_for_status(lib().card_pfwd_bind(self.h, ptr(rows.pos), ptr(rows.slot)), "card_pfwd_bind")

    def run(self, dM: torch.Tensor, step_begin: int, step_end: int):
        raise_for_status(lib().card_pfwd_run(self.h, ptr(dM), step_begin, step_end, stream_ptr()), "card_pfwd_run")

    def info(self) -> dict:
        buf = (ctypes.c_int32 * 16)()
        lib().card_pfwd_info(self.h, ctypes.cast(buf, ctypes.c_void_p))
        names = ("qkv", "attn", "o", "gu", "d")
        return {"grid": buf[0], "smem": buf[1], "w_stages": buf[2], "x_stages": buf[3], "Mpad": buf[4],
                "splits": {names[p]: buf[5 + 2 * p] for p in range(5) if p != 1}, "worker_groups": buf[15]}

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().card_pfwd_destroy(self.h)
        except Exception:
            pass


class DeviceLlama:
    """One draft or target model resident in HBM with its KV cache.

    ``plans`` are per row-budget (e.g. 1 for AR decode, r+1 for verify,
    K+max_depth+2 for draft tree steps, 128 for prefill chunks); each plan
    owns the GEMM launch configurations (tensor maps, split-K workspaces)
    bound to the shared activation buffers.
    """

    def __init__(self, cfg: LlamaConfig, packed: dict, *, max_ctx: int, tree_slots: int = 0,
                 row_budgets=(1,), extra_max: int = 32, tp=None, pool_requests: int = 8,
                 persistent: bool = True):
        """tp: (comm, shards, full_vocab) of a tensor-parallel target rank (tp.py):
        cfg is then the rank's shard; o / down write partials that are
        all-reduced before the residual add, and the vocabulary slices of
        the lm_head are summed into full-vocabulary logits."""
        self.dev = require_cuda()
        self.tp = tp
        # wide row budgets (draft tree steps) run the persistent forward (_PFwd)
        self.persistent = persistent
        dtype = packed["dtype"]
        self.cfg = cfg
        self.dtype = dtype
        self.wdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.code = 0 if dtype == "bf16" else 1
        self.max_ctx = max_ctx
        self.prefix_slots = ((max_ctx + 63) // 64) * 64      # longest context (logical positions)
        # paged prefix KV (bf16 path): a pool for pool_requests contexts, handed
        # out page by page to the requests on this runtime (PagePool)
        self.pool_pages = (self.prefix_slots // PAGE) * pool_requests
        self.page_pool = PagePool(self.pool_pages)
        self.tree_base = self.pool_pages * PAGE
        self.n_slots = self.tree_base + tree_slots
        self.tree_slots = tree_slots
        self.extra_max = extra_max
        c = cfg
        dev = self.dev
        wdt = self.wdt
        H, hd = c.hidden, c.head_dim
        self.embed = packed["embed"]
        self.lm_head = packed["lm_head"]
        self.norm = packed["norm"]
        self.layers = packed["layers"]
        kvdt = wdt
        self.k_cache = [torch.zeros((self.n_slots, c.n_kv_heads, hd), dtype=kvdt, device=dev) for _ in range(c.n_layers)]
        self.v_cache = [torch.zeros((self.n_slots, c.n_kv_heads, hd), dtype=kvdt, device=dev) for _ in range(c.n_layers)]
        cos, sin = rope_tables(c, max_ctx + 8)
        self.cos, self.sin = cos.to(dev), sin.to(dev)
        # activation buffers sized for the largest row budget
        mmax = max(row_budgets)
        self.mpad = ((mmax + 15) // 16) * 16
        act = wdt
        P = self.mpad
        self.x = torch.zeros((P, H), dtype=torch.float32, device=dev)
        self.h = torch.zeros((P, H), dtype=act, device=dev)
        self.qkv = torch.zeros((P, c.qkv_dim), dtype=torch.float32, device=dev)
        self.q = torch.zeros((P, c.n_heads * hd), dtype=torch.float32, device=dev)
        self.o = torch.zeros((P, c.n_heads * hd), dtype=act, device=dev)
        self.g = torch.zeros((P, c.ffn), dtype=act, device=dev)
        self.hf = torch.zeros((P, H), dtype=act, device=dev)
        self.logits = torch.zeros((P, c.vocab_size), dtype=torch.float32, device=dev)
        if tp is not None:
            comm, shards, V_full = tp
            self.tp_vocab = shards[comm.rank].vocab
            self.logits_local = self.logits                        # [P, this rank's padded slice]
            self.logits = torch.zeros((P, V_full), dtype=torch.float32, device=dev)
            self.part = torch.zeros((P, H), dtype=torch.float32, device=dev)
        # fused-norm path (bf16): bf16 residual copy + per-16-column sums of squares
        self.fused = bool(packed.get("folded")) and H % 16 == 0 and hd in (64, 128) and \
            (c.qkv_dim % 128 == 0) and (c.n_heads * hd) % 128 == 0 and (c.n_kv_heads * hd) % 128 == 0
        self.xb = torch.zeros((P, H), dtype=torch.bfloat16, device=dev) if self.fused else None
        self.ssq = torch.zeros((H // 16, P), dtype=torch.float32, device=dev) if self.fused else None
        nwork = lib().card_attention_work_floats(P, c.n_heads, hd, self.prefix_slots)
        self.work = torch.zeros(nwork, dtype=torch.float32, device=dev)
        # per-layer KV base pointer arrays for the engine's KV movers
        self.k_ptrs = torch.tensor([t.data_ptr() for t in self.k_cache], dtype=torch.int64, device=dev)
        self.v_ptrs = torch.tensor([t.data_ptr() for t in self.v_cache], dtype=torch.int64, device=dev)
        if tp is not None and not self.fused:
            raise ConfigError("the tensor-parallel target runs the fused bf16 path (head_dim 64/128, 128-aligned shards)")
        self.rows_placeholder = torch.zeros(P, dtype=torch.int32, device=dev)
        self.plans = {m: self._make_plan(m) for m in sorted(set(row_budgets))}

    # ------------------------------------------------------------ plans
    def _make_plan(self, m_max: int) -> dict:
        if self.fused:
            return self._make_fused_plan(m_max)
        c = self.cfg
        H = c.hidden
        plan = {"m_max": m_max, "layers": []}
        for L in self.layers:
            plan["layers"].append({
                "qkv": _Linear(L["wqkv"], self.h, m_max, EPI_STORE_F32, self.qkv, c.qkv_dim, L["bqkv"]),
                "o": _Linear(L["wo"], self.o, m_max, EPI_RESID_F32, self.x, H),
                "gu": _Linear(L["wgu"], self.h, m_max, EPI_SWIGLU_BF16, self.g, c.ffn),
                "d": _Linear(L["wd"], self.g, m_max, EPI_RESID_F32, self.x, H),
            })
        plan["lm_head"] = _Linear(self.lm_head, self.hf, m_max, EPI_STORE_F32, self.logits, c.vocab_size)
        return plan

    def _make_fused_plan(self, m_max: int) -> dict:
        """bf16: 5 kernels per layer — qkv (+RMSNorm scale, RoPE, KV write),
        attention, o (+residual, +sum of squares), gate/up (+RMSNorm scale,
        SwiGLU), down (+residual, +sum of squares)."""
        c = self.cfg
        H, P = c.hidden, self.mpad
        parts = H // 16
        plan = {"m_max": m_max, "layers": [], "bound_rows": None}
        for li, L in enumerate(self.layers):
            qkv = _Linear(L["wqkv"], self.xb, m_max, EPI_QKV_ROPE, self.qkv, c.qkv_dim, L["bqkv"])
            qkv.fuse_norm(self.ssq, parts, P, c.rms_eps, H)
            if self.tp is None:
                o = _Linear(L["wo"], self.o, m_max, EPI_RESID_F32, self.x, H)
                o.fuse_resid(self.ssq, P, self.xb)
            else:   # row-parallel: partial -> all-reduce -> card_resid_add
                o = _Linear(L["wo"], self.o, m_max, EPI_STORE_F32, self.part, H)
            gu = _Linear(L["wgu"], self.xb, m_max, EPI_SWIGLU_BF16, self.g, c.ffn)
            gu.fuse_norm(self.ssq, parts, P, c.rms_eps, H)
            if self.tp is None:
                d = _Linear(L["wd"], self.g, m_max, EPI_RESID_F32, self.x, H)
                d.fuse_resid(self.ssq, P, self.xb)
            else:
                d = _Linear(L["wd"], self.g, m_max, EPI_STORE_F32, self.part, H)
            plan["layers"].append({"qkv": qkv, "o": o, "gu": gu, "d": d})
        plan["lm_head"] = _Linear(self.lm_head, self.xb, m_max, EPI_STORE_F32,
                                  self.logits if self.tp is None else self.logits_local, c.vocab_size)
        # (narrow plans — verify, AR — keep the per-GEMM kernels: a persistent
        # M = 8 verify of Llama-3.1-8B measured 4.03 vs 3.31 ms, tools/pfwd_target_probe.py)
        if self.persistent and self.tp is None and 16 < m_max <= 128:
            plan["pfwd"] = _PFwd(self, m_max)
        return plan

    def _tp_reduce(self, dM, mm):
        """All-reduce the row-parallel partial, then x += part (+ bf16 copy, ssq)."""
        comm = self.tp[0]
        comm.all_reduce(self.part)
        raise_for_status(lib().card_resid_add(ptr(dM), mm, self.cfg.hidden, ptr(self.x), ptr(self.part), ptr(self.xb),
                                              ptr(self.ssq), self.mpad, stream_ptr()), "card_resid_add")

    def _tp_gather_logits(self):
        """Vocabulary slices -> full logits on every rank: each rank writes its
        slice into zeros and an all-reduce sums them (exact: x + 0 = x)."""
        comm = self.tp[0]
        v0, v1 = self.tp_vocab
        self.logits.zero_()
        self.logits[:, v0:v1].copy_(self.logits_local[:, :v1 - v0])
        comm.all_reduce(self.logits)

    def _bind_rows(self, plan: dict, rows: "RowBlock"):
        """Row-dependent epilogue pointers (positions, KV slots, lm_head row offset)."""
        key = rows.block.data_ptr()
        if plan.get("bound_rows") == key:
            return
        c = self.cfg
        for li, P_ in enumerate(plan["layers"]):
            P_["qkv"].fuse_rope(rows, self.cos, self.sin, c.n_heads, c.n_kv_heads, c.head_dim, self.q,
                                self.k_cache[li], self.v_cache[li])
        plan["lm_head"].fuse_norm(self.ssq, c.hidden // 16, self.mpad, c.rms_eps, c.hidden, rows.out_rows)
        if "pfwd" in plan:
            plan["pfwd"].bind(rows)
        if "lm_head_topk" in plan:
            plan["lm_head_topk"].fuse_norm(self.ssq, c.hidden // 16, self.mpad, c.rms_eps, c.hidden, rows.out_rows)
        plan["bound_rows"] = key

    def kv_row_elems(self) -> int:
        return self.cfg.n_kv_heads * self.cfg.head_dim

    def kv_esize(self) -> int:
        return 2 if self.dtype == "bf16" else 4

    # ------------------------------------------------------------ forward
    def page_table(self, device=None) -> "PageTable | None":
        """Pages for one request's context (bf16 path); None on the fp32 parity
        path, which addresses its KV by position."""
        if not self.fused:
            return None
        return PageTable(self.page_pool, self.prefix_slots // PAGE, device or self.dev)

    def forward(self, rows: "RowBlock", m_max: int, topk: bool = False, pages: "PageTable | None" = None,
                batch: "BatchPages | None" = None, head: bool = True):
        """Run the forward over the device rows; logits for the output rows
        land in self.logits[:n_out] (topk=True: the lm_head_topk records
        instead, see lm_topk_head).  pages: the request's page table (the
        rows' KV slots were built through it); None = identity.
        Asynchronous, graph-capturable."""
        c = self.cfg
        L_ = lib()
        s = stream_ptr()
        plan = self.plans[m_max]
        if self.fused:
            return self._forward_fused(rows, plan, topk, pages, batch, head)
        if topk:
            raise ConfigError("the fused top-k lm_head needs the bf16 path")
        if batch is not None:
            raise ConfigError("batched forwards run the bf16 paged path")
        dM, dOut = rows.M, rows.n_out
        hd = c.head_dim
        mm = plan["m_max"]   # grids sized for this plan's rows (rows >= M exit at once)
        chk = raise_for_status
        chk(L_.card_embed(ptr(rows.tok), ptr(dM), mm, ptr(self.embed), self.code, c.hidden, ptr(self.x), None, None, 0, s),
            "embed")
        for li, (L, P) in enumerate(zip(self.layers, plan["layers"])):
            chk(L_.card_rmsnorm(ptr(self.x), ptr(L["attn_norm"]), c.hidden, c.rms_eps, ptr(dM), mm, None,
                                ptr(self.h), self.code, s), "rmsnorm")
            P["qkv"].run(dM)
            chk(L_.card_rope_kv(ptr(self.qkv), ptr(dM), mm, ptr(rows.pos), ptr(rows.slot), ptr(self.cos),
                                ptr(self.sin), c.n_heads, c.n_kv_heads, hd, ptr(self.q), ptr(self.k_cache[li]),
                                ptr(self.v_cache[li]), self.code, s), "rope_kv")
            chk(L_.card_attention(ptr(self.q), ptr(dM), mm, ptr(rows.plen), ptr(rows.slot), ptr(rows.n_extra), ptr(rows.extra),
                                  rows.extra_max, ptr(self.k_cache[li]), ptr(self.v_cache[li]), self.code,
                                  c.n_heads, c.n_kv_heads, hd, self.prefix_slots, ptr(self.work), ptr(self.o),
                                  self.code, s), "attention")
            P["o"].run(dM)
            chk(L_.card_rmsnorm(ptr(self.x), ptr(L["mlp_norm"]), c.hidden, c.rms_eps, ptr(dM), mm, None,
                                ptr(self.h), self.code, s), "rmsnorm")
            P["gu"].run(dM)
            P["d"].run(dM)
        chk(L_.card_rmsnorm(ptr(self.x), ptr(self.norm), c.hidden, c.rms_eps, ptr(dOut), mm, ptr(rows.out_rows),
                            ptr(self.hf), self.code, s), "final norm")
        plan["lm_head"].run(dOut)

    def lm_topk_head(self, m_max: int):
        """The fused lm_head + softmax + top-k linear of plan m_max (bf16 path;
        None on the fp32 path): EPI_TOPK records instead of logits, merged by
        card_lmhead_topk_merge.  Built on first use."""
        if not self.fused:
            return None
        plan = self.plans[m_max]
        lin = plan.get("lm_head_topk")
        if lin is None:
            n_tiles = self.lm_head.shape[0] if self.lm_head.dim() == 4 else self.lm_head.shape[0] // 128
            work = torch.zeros(m_max * n_tiles * TOPK_REC, dtype=torch.float32, device=self.dev)
            lin = _Linear(self.lm_head, self.xb, m_max, EPI_TOPK, work, 0)
            lin.work, lin.n_tiles = work, n_tiles
            plan["lm_head_topk"] = lin
            plan["bound_rows"] = None   # rebind the row offset of the new head
        return lin

    def _attend(self, li: int, rows: "RowBlock", mm: int, pages, batch, qsw=None, qsw_tiles: int = 0):
        """Attention of layer li over the row block: one request's paged KV
        (pages), or several requests' (batch: each row region its own table)."""
        c = self.cfg
        L_ = lib()
        if batch is not None:
            return raise_for_status(L_.card_attention_batch(
                None if qsw is not None else ptr(self.q), ptr(qsw), qsw_tiles, ptr(rows.M), mm, ptr(rows.plen),
                ptr(rows.n_extra), ptr(rows.extra), rows.extra_max, ptr(self.k_cache[li]), ptr(self.v_cache[li]),
                ptr(batch.tables), batch.stride, batch.seg_rows, c.n_heads, c.n_kv_heads, c.head_dim,
                self.prefix_slots, ptr(self.o), stream_ptr()), "attention (batch)")
        pt = ptr(pages.dev) if pages is not None else None
        if qsw is not None:
            return raise_for_status(L_.card_attention_tree(
                ptr(qsw), qsw_tiles, ptr(rows.M), mm, ptr(rows.plen), ptr(rows.n_extra), ptr(rows.extra),
                rows.extra_max, ptr(self.k_cache[li]), ptr(self.v_cache[li]), pt, c.n_heads, c.n_kv_heads,
                c.head_dim, self.prefix_slots, ptr(self.o), stream_ptr()), "attention")
        return raise_for_status(L_.card_attention_paged(
            ptr(self.q), ptr(rows.M), mm, ptr(rows.plen), ptr(rows.n_extra), ptr(rows.extra), rows.extra_max,
            ptr(self.k_cache[li]), ptr(self.v_cache[li]), pt, c.n_heads, c.n_kv_heads, c.head_dim,
            self.prefix_slots, ptr(self.o), stream_ptr()), "attention")

    def _forward_fused(self, rows: "RowBlock", plan: dict, topk: bool = False, pages: "PageTable | None" = None,
                       batch: "BatchPages | None" = None, head: bool = True):
        """head=False stops before the lm_head (its input rows: xb / ssq at
        the rows' out_rows, e.g. for card_gather_rows)."""
        c = self.cfg
        L_ = lib()
        s = stream_ptr()
        self._bind_rows(plan, rows)
        dM = rows.M
        mm = plan["m_max"]
        chk = raise_for_status
        chk(L_.card_embed(ptr(rows.tok), ptr(dM), mm, ptr(self.embed), self.code, c.hidden, ptr(self.x), ptr(self.xb),
                          ptr(self.ssq), self.mpad, s), "embed")
        pf = plan.get("pfwd")
        if pf is not None:
            n5 = _PFwd.PHASES
            # wide row blocks read Q pre-swizzled by the tcgen05 attention; narrow
            # ones (verify, AR) keep fp32 q for the register-resident kernel
            tree_q = pf.use_qsw(rows.extra_max if mm * (c.n_heads // c.n_kv_heads) >= 256 else 1 << 30)
            pf.run(dM, 0, 1)   # layer 0 qkv
            for li in range(c.n_layers):
                self._attend(li, rows, mm, pages, batch, pf.qsw if tree_q else None, pf.qsw_tiles if tree_q else 0)
                # o, gate/up, down of layer li, then the qkv of layer li + 1
                pf.run(dM, n5 * li + 2, min(n5 * (li + 1) + 1, n5 * c.n_layers))
            if head:
                plan["lm_head_topk" if topk else "lm_head"].run(rows.n_out)
            return
        for li, P in enumerate(plan["layers"]):
            P["qkv"].run(dM)
            self._attend(li, rows, mm, pages, batch)
            P["o"].run(dM)
            if self.tp is not None:
                self._tp_reduce(dM, mm)
            P["gu"].run(dM)
            P["d"].run(dM)
            if self.tp is not None:
                self._tp_reduce(dM, mm)
        if not head:
            return
        plan["lm_head_topk" if topk else "lm_head"].run(rows.n_out)
        if self.tp is not None:
            if topk:
                raise ConfigError("the fused top-k lm_head is a draft path; a tensor-parallel target gathers logits")
            self._tp_gather_logits()

    def launches_per_forward(self) -> int:
        gu_extra = 0
        return 2 + self.cfg.n_layers * (2 + 1 + 1 + 3 + 1 + 1 + 1 + gu_extra) + 2


@dataclass
class BatchPages:
    """Page tables of the requests of a batched forward: request i owns rows
    [i * seg_rows, (i + 1) * seg_rows) and its prefix page table is
    tables[i] (int32 [B, stride] on the device)."""
    tables: torch.Tensor
    stride: int
    seg_rows: int


class RowBlock:
    """Device row descriptors (see csrc/card_llm.h CardRows): one int32 block
    [M, n_out, tok, pos, slot, plen, n_extra, out_rows, extra]."""

    def __init__(self, rows_max: int, extra_max: int, device):
        self.rows_max = rows_max
        self.extra_max = extra_max
        R = rows_max
        self.block = torch.zeros(2 + 6 * R + R * extra_max, dtype=torch.int32, device=device)
        b = self.block
        self.M = b[0:1]
        self.n_out = b[1:2]
        self.tok = b[2:2 + R]
        self.pos = b[2 + R:2 + 2 * R]
        self.slot = b[2 + 2 * R:2 + 3 * R]
        self.plen = b[2 + 3 * R:2 + 4 * R]
        self.n_extra = b[2 + 4 * R:2 + 5 * R]
        self.out_rows = b[2 + 5 * R:2 + 6 * R]
        self.extra = b[2 + 6 * R:]

    def set_chain(self, tokens, start_pos: int, out_last_only=True, pages: "PageTable | None" = None) -> int:
        """Host helper: causal chain rows (prefill / AR decode), KV slots
        through the request's page table; returns the bytes copied to the
        device."""
        n = len(tokens)
        assert n <= self.rows_max
        host = torch.zeros(2 + 6 * self.rows_max, dtype=torch.int32)
        R = self.rows_max
        host[0] = n
        host[1] = 1 if out_last_only else n
        host[2:2 + n] = torch.tensor(tokens, dtype=torch.int32)
        pos = torch.arange(start_pos, start_pos + n, dtype=torch.int32)
        host[2 + R:2 + R + n] = pos
        host[2 + 2 * R:2 + 2 * R + n] = pos if pages is None else \
            torch.tensor([pages.slot(p) for p in range(start_pos, start_pos + n)], dtype=torch.int32)
        host[2 + 3 * R:2 + 3 * R + n] = pos + 1
        if out_last_only:
            host[2 + 5 * R] = n - 1
        else:
            host[2 + 5 * R:2 + 5 * R + n] = torch.arange(n, dtype=torch.int32)
        self.block[: 2 + 6 * R].copy_(host, non_blocking=False)
        return host.numel() * 4   # host->device bytes
