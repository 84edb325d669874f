"""CPU fp32 tensor-parallel restatement of oracle/llama_ref.py — TEST
INFRASTRUCTURE ONLY.

Runs one rank's share of the forward from ``paper_2508_04462_b200.tp``
shard weights: local q/k/v heads and attention, row-parallel o and down
partials summed with an all-reduce, vocab-parallel lm_head gathered into
the full vocabulary.  tests/test_tp.py runs it under gloo with world size 2
and 3 and compares the gathered logits with the unsharded RefLlama.
"""

from __future__ import annotations

import math

import torch

from oracle.llama_ref import inv_freq


def tp_forward(cfg, shards, rank: int, w: dict, tokens: list[int], comm) -> torch.Tensor:
    """Full-context logits [n, V] of ``tokens`` on this rank (identical on all)."""
    shard = shards[rank]
    n = len(tokens)
    nh = shard.q_heads[1] - shard.q_heads[0]
    nkv = shard.kv_heads[1] - shard.kv_heads[0]
    hd = cfg.head_dim
    G = cfg.n_heads // cfg.n_kv_heads
    inv = inv_freq(cfg)
    pos = torch.arange(n)
    freqs = torch.outer(pos.float(), inv)
    cos, sin = freqs.cos()[:, None, :], freqs.sin()[:, None, :]

    def rope(x):
        h = x.shape[-1] // 2
        return torch.cat([x[..., :h] * cos - x[..., h:] * sin, x[..., h:] * cos + x[..., :h] * sin], dim=-1)

    def rms(x, wt):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + cfg.rms_eps) * wt

    f = {k: v.float() for k, v in w.items()}
    x = f["embed"][torch.tensor(tokens)]
    causal = torch.arange(n)[None, :] > pos[:, None]
    for i in range(cfg.n_layers):
        p = f"l{i}."
        h = rms(x, f[p + "attn_norm"])
        q = rope((h @ f[p + "wq"].T).view(n, nh, hd))
        k = rope((h @ f[p + "wk"].T).view(n, nkv, hd))
        v = (h @ f[p + "wv"].T).view(n, nkv, hd)
        kx, vx = k.repeat_interleave(G, dim=1), v.repeat_interleave(G, dim=1)
        s = torch.einsum("nhd,thd->hnt", q, kx) / math.sqrt(hd)
        a = torch.softmax(s.masked_fill(causal[None], float("-inf")), dim=-1)
        o = torch.einsum("hnt,thd->nhd", a, vx).reshape(n, nh * hd)
        part = o @ f[p + "wo"].T
        comm.all_reduce(part)
        x = x + part
        h = rms(x, f[p + "mlp_norm"])
        part = (torch.nn.functional.silu(h @ f[p + "wg"].T) * (h @ f[p + "wu"].T)) @ f[p + "wd"].T
        comm.all_reduce(part)
        x = x + part
    local = rms(x, f["norm"]) @ f["lm_head"].T          # [n, vocab_padded]
    parts = [torch.zeros_like(local) for _ in range(comm.world)]
    comm.all_gather(parts, local.contiguous())
    return torch.cat([pc[:, :sh.vocab[1] - sh.vocab[0]] for pc, sh in zip(parts, shards)], dim=1)
