"""Tensor-parallel target model (BASELINE configs[3]: Llama-3.1-70B over 7
GPUs).

Megatron-style split of one transformer over ``world`` ranks, uneven where
the shapes do not divide:

* attention: whole GQA groups per rank — kv heads split as evenly as
  possible (8 kv heads over 7 ranks: 2, 1, 1, 1, 1, 1, 1), each rank holding
  the q heads of its kv heads; QKV column-parallel (its head rows), o
  row-parallel (its head columns) followed by an all-reduce of the partial;
* MLP: gate/up column-parallel over 64-row units of the FFN, down
  row-parallel, all-reduce;
* lm_head: vocab-parallel over 128-row tiles (1002 tiles over 7 ranks:
  144 / 143 each), the last shard zero-padded to a whole tile; the logits
  are all-gathered into the full vocabulary before argmax / softmax;
* embedding, norms and the residual stream are replicated: after each
  all-reduce every rank holds the same fp32 residual.

A rank's shard is itself a (narrower) Llama config, so the device forward,
the fused GEMM epilogues and the attention run unchanged on it; only the o
and down projections write a partial that ``DeviceLlama`` reduces with the
communicator (NCCL over NVLink in production, gloo in the CPU tests).
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import torch

from .errors import ConfigError

VOCAB_TILE = 128
FFN_UNIT = 64


@dataclass(frozen=True)
class TPShard:
    rank: int
    world: int
    kv_heads: tuple[int, int]   # [lo, hi) kv heads
    q_heads: tuple[int, int]    # [lo, hi) q heads (the GQA groups of kv_heads)
    ffn: tuple[int, int]        # [lo, hi) FFN features
    vocab: tuple[int, int]      # [lo, hi) vocabulary rows (real, unpadded)
    vocab_padded: int           # rows of this rank's lm_head (multiple of 128)


def _split(n: int, world: int) -> list[tuple[int, int]]:
    base, extra = divmod(n, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def tp_shards(cfg, world: int) -> list[TPShard]:
    """Per-rank head / FFN / vocabulary ranges (uneven splits allowed)."""
    if world < 1:
        raise ConfigError("tensor-parallel world size must be >= 1")
    if cfg.n_kv_heads < world:
        raise ConfigError(f"{cfg.n_kv_heads} kv heads cannot be split over {world} ranks (whole GQA groups per rank)")
    if cfg.ffn % FFN_UNIT:
        raise ConfigError(f"ffn {cfg.ffn} is not a multiple of {FFN_UNIT}")
    G = cfg.n_heads // cfg.n_kv_heads
    kv = _split(cfg.n_kv_heads, world)
    ff = _split(cfg.ffn // FFN_UNIT, world)
    n_tiles = -(-cfg.vocab_size // VOCAB_TILE)
    vt = _split(n_tiles, world)
    if min(hi - lo for lo, hi in ff) < 1 or min(hi - lo for lo, hi in vt) < 1:
        raise ConfigError(f"FFN or vocabulary too small for {world} ranks")
    out = []
    for r in range(world):
        v0, v1 = vt[r][0] * VOCAB_TILE, min(cfg.vocab_size, vt[r][1] * VOCAB_TILE)
        out.append(TPShard(r, world, kv[r], (kv[r][0] * G, kv[r][1] * G),
                           (ff[r][0] * FFN_UNIT, ff[r][1] * FFN_UNIT), (v0, v1),
                           (vt[r][1] - vt[r][0]) * VOCAB_TILE))
    return out


def shard_config(cfg, sh: TPShard):
    """The rank's slice as a Llama config (its heads, FFN and vocabulary)."""
    return dataclasses.replace(cfg, vocab_size=sh.vocab_padded, n_heads=sh.q_heads[1] - sh.q_heads[0],
                               n_kv_heads=sh.kv_heads[1] - sh.kv_heads[0], ffn=sh.ffn[1] - sh.ffn[0],
                               tie_embeddings=False)


def shard_weights(cfg, weights: dict, sh: TPShard) -> dict:
    """Canonical (llama.init_weights layout) weights of one rank.  The full
    embedding stays on every rank (token lookup); lm_head keeps the rank's
    vocabulary rows, zero-padded to a whole 128-row tile."""
    hd = cfg.head_dim
    q0, q1 = sh.q_heads[0] * hd, sh.q_heads[1] * hd
    k0, k1 = sh.kv_heads[0] * hd, sh.kv_heads[1] * hd
    f0, f1 = sh.ffn
    out = {"embed": weights["embed"], "norm": weights["norm"]}
    for i in range(cfg.n_layers):
        p = f"l{i}."
        out[p + "wq"] = weights[p + "wq"][q0:q1].contiguous()
        out[p + "wk"] = weights[p + "wk"][k0:k1].contiguous()
        out[p + "wv"] = weights[p + "wv"][k0:k1].contiguous()
        if cfg.qkv_bias:
            out[p + "bq"] = weights[p + "bq"][q0:q1].contiguous()
            out[p + "bk"] = weights[p + "bk"][k0:k1].contiguous()
            out[p + "bv"] = weights[p + "bv"][k0:k1].contiguous()
        out[p + "wo"] = weights[p + "wo"][:, q0:q1].contiguous()
        out[p + "wg"] = weights[p + "wg"][f0:f1].contiguous()
        out[p + "wu"] = weights[p + "wu"][f0:f1].contiguous()
        out[p + "wd"] = weights[p + "wd"][:, f0:f1].contiguous()
        out[p + "attn_norm"] = weights[p + "attn_norm"]
        out[p + "mlp_norm"] = weights[p + "mlp_norm"]
    head = weights["lm_head"][sh.vocab[0]:sh.vocab[1]]
    pad = sh.vocab_padded - head.shape[0]
    if pad:
        head = torch.cat([head, torch.zeros(pad, head.shape[1], dtype=head.dtype, device=head.device)])
    out["lm_head"] = head.contiguous()
    return out


def shard_stream(cfg, items, sh: TPShard) -> dict:
    """shard_weights over a (name, tensor) stream (llama.iter_weights): each
    full tensor is sliced as it is produced, so a rank of a 70B target never
    holds more than one full matrix at a time."""
    hd = cfg.head_dim
    rows = {"wq": (sh.q_heads[0] * hd, sh.q_heads[1] * hd), "wk": (sh.kv_heads[0] * hd, sh.kv_heads[1] * hd),
            "bq": (sh.q_heads[0] * hd, sh.q_heads[1] * hd), "bk": (sh.kv_heads[0] * hd, sh.kv_heads[1] * hd),
            "wg": sh.ffn, "wu": sh.ffn}
    rows["wv"], rows["bv"] = rows["wk"], rows["bk"]
    cols = {"wo": (sh.q_heads[0] * hd, sh.q_heads[1] * hd), "wd": sh.ffn}
    out = {}
    for name, t in items:
        key = name.split(".")[-1]
        if key in rows:
            lo, hi = rows[key]
            out[name] = t[lo:hi].contiguous()
        elif key in cols:
            lo, hi = cols[key]
            out[name] = t[:, lo:hi].contiguous()
        elif name == "lm_head":
            out[name] = t[sh.vocab[0]:sh.vocab[1]].contiguous()
        else:
            out[name] = t
        del t
    if "lm_head" not in out:   # tied: the embedding rows
        out["lm_head"] = out["embed"][sh.vocab[0]:sh.vocab[1]].contiguous()
    head = out["lm_head"]
    pad = sh.vocab_padded - head.shape[0]
    if pad:
        out["lm_head"] = torch.cat([head, torch.zeros(pad, head.shape[1], dtype=head.dtype, device=head.device)])
    return out


class TPComm:
    """The collectives a tensor-parallel forward needs, over a
    torch.distributed process group (NCCL across GPUs; gloo works too)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_reduce(self, t: torch.Tensor) -> None:
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def all_gather(self, out: list[torch.Tensor], t: torch.Tensor) -> None:
        self.dist.all_gather(out, t, group=self.group)
