"""CPU fp32 Llama-architecture oracle — TEST INFRASTRUCTURE ONLY.

The reference contains no transformer ("transformer
arithmetic ... parity unpinned" in the reference itself).  This is an
independent torch-CPU restatement of the Llama/Qwen2 forward (RMSNorm,
RoPE with Llama-3 scaling, GQA attention, SwiGLU), pinned against HF
``transformers`` ``LlamaForCausalLM`` in tests/test_oracle_llama.py.  It
plugs into the reference's model protocol (``next_distribution``,
lm.py:140-153) so the reference engine — or its oracle restatement in
card_oracle.run_serial — can drive it unchanged.

Only tests/, smoke() and bench.py's CPU-baseline legs may use it.
"""

from __future__ import annotations

import math

import numpy as np
import torch


def inv_freq(cfg) -> torch.Tensor:
    hd = cfg.head_dim
    base = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.int64).float() / hd))
    sc = cfg.rope_scaling
    if not sc:
        return base
    factor, lo, hi, old = (sc["factor"], sc["low_freq_factor"], sc["high_freq_factor"],
                           sc["original_max_position_embeddings"])
    out = []
    for f in base.tolist():
        wl = 2 * math.pi / f
        if wl < old / hi:
            out.append(f)
        elif wl > old / lo:
            out.append(f / factor)
        else:
            s = (old / wl - lo) / (hi - lo)
            out.append((1 - s) * f / factor + s * f)
    return torch.tensor(out, dtype=torch.float32)


class RefLlama:
    """fp32 CPU forward with an incremental KV cache over one token stream."""

    def __init__(self, cfg, weights: dict, threads: int | None = None):
        self.cfg = cfg
        self.w = {k: v.detach().to("cpu", torch.float32) for k, v in weights.items()}
        self.inv = inv_freq(cfg)
        if threads:
            torch.set_num_threads(threads)
        self.tokens: list[int] = []
        self.kv: list[tuple[torch.Tensor, torch.Tensor]] = []
        self.last_logits: torch.Tensor | None = None

    # ------------------------------------------------------------ pieces
    def _rms(self, x, w):
        var = x.pow(2).mean(-1, keepdim=True)
        return (x * torch.rsqrt(var + self.cfg.rms_eps)) * w

    def _rope(self, x, pos):
        # x [n, heads, hd]; rotate_half convention
        freqs = torch.outer(pos.float(), self.inv)            # [n, hd/2]
        cos, sin = freqs.cos()[:, None, :], freqs.sin()[:, None, :]
        h = x.shape[-1] // 2
        x1, x2 = x[..., :h], x[..., h:]
        return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)

    def _extend(self, new_tokens: list[int], out: str = "all") -> torch.Tensor | None:
        """Append tokens to the cached stream; returns logits [n_new, V]
        (out="all"), of the last token only [1, V] ("last"), or None."""
        c = self.cfg
        n0 = len(self.tokens)
        n = len(new_tokens)
        pos = torch.arange(n0, n0 + n)
        x = self.w["embed"][torch.tensor(new_tokens)]
        nh, nkv, hd = c.n_heads, c.n_kv_heads, c.head_dim
        g = nh // nkv
        for i in range(c.n_layers):
            p = f"l{i}."
            h = self._rms(x, self.w[p + "attn_norm"])
            q = h @ self.w[p + "wq"].T
            k = h @ self.w[p + "wk"].T
            v = h @ self.w[p + "wv"].T
            if c.qkv_bias:
                q, k, v = q + self.w[p + "bq"], k + self.w[p + "bk"], v + self.w[p + "bv"]
            q = self._rope(q.view(n, nh, hd), pos)
            k = self._rope(k.view(n, nkv, hd), pos)
            v = v.view(n, nkv, hd)
            if len(self.kv) <= i:
                self.kv.append((k, v))
            else:
                pk, pv = self.kv[i]
                self.kv[i] = (torch.cat([pk[:n0], k]), torch.cat([pv[:n0], v]))
            K, V = self.kv[i]
            Kx = K.repeat_interleave(g, dim=1)                 # [T, nh, hd]
            Vx = V.repeat_interleave(g, dim=1)
            s = torch.einsum("nhd,thd->hnt", q, Kx) / math.sqrt(hd)
            T = K.shape[0]
            mask = torch.arange(T)[None, :] > (pos[:, None])
            s = s.masked_fill(mask[None], float("-inf"))
            a = torch.softmax(s, dim=-1)
            o = torch.einsum("hnt,thd->nhd", a, Vx).reshape(n, nh * hd)
            x = x + o @ self.w[p + "wo"].T
            h = self._rms(x, self.w[p + "mlp_norm"])
            gg = h @ self.w[p + "wg"].T
            uu = h @ self.w[p + "wu"].T
            x = x + (torch.nn.functional.silu(gg) * uu) @ self.w[p + "wd"].T
        self.tokens.extend(int(t) for t in new_tokens)
        if out == "none":
            return None
        if out == "last":
            x = x[-1:]
        x = self._rms(x, self.w["norm"])
        return x @ self.w["lm_head"].T

    def logits_for(self, context: list[int]) -> torch.Tensor:
        """Logits after `context`: reuses the cached common prefix."""
        ctx = [int(t) for t in context]
        c = 0
        m = min(len(ctx), len(self.tokens))
        while c < m and ctx[c] == self.tokens[c]:
            c += 1
        if c == len(ctx):      # context is a prefix of the cache: recompute its last token
            c -= 1
        self.tokens = self.tokens[:c]
        self.kv = [(k[:c], v[:c]) for k, v in self.kv]
        return self._extend(ctx[c:])[-1]

    def full_logits(self, tokens: list[int]) -> torch.Tensor:
        self.tokens, self.kv = [], []
        return self._extend(list(tokens))

    # ------------------------------------------------------------ batched passes
    def _sync(self, prefix: list[int]) -> None:
        """Make the cached stream exactly `prefix` (reuse the common part)."""
        c, m = 0, min(len(prefix), len(self.tokens))
        while c < m and prefix[c] == self.tokens[c]:
            c += 1
        self.tokens = self.tokens[:c]
        self.kv = [(k[:c], v[:c]) for k, v in self.kv]
        if c < len(prefix):
            self._extend(prefix[c:], "none")

    def chain_logits(self, ctx: list[int], toks: list[int]) -> torch.Tensor:
        """Logits after ctx + toks[:i] for i = 0..len(toks): one pass over
        the chain (a verify's rows) instead of len(toks) + 1 extensions."""
        ctx = [int(t) for t in ctx]
        self._sync(ctx[:-1])
        return self._extend([ctx[-1]] + [int(t) for t in toks], "all")

    def tree_logits(self, base: list[int], paths: list[list[int]]) -> torch.Tensor:
        """Logits after base + path for each path: one masked pass over the
        newest tree layer (each row's last token), attending to the cached
        base stream plus its ancestors' keys, which are kept per node (keyed
        by the node's full context) from the layers that produced them."""
        base = [int(t) for t in base]
        self._sync(base)
        if not hasattr(self, "node_kv") or len(self.node_kv) > 50000:
            self.node_kv = {}
        nb = len(base)
        for key in [k for k in self.node_kv if len(k) <= nb]:   # now part of the stream
            del self.node_kv[key]
        bt = tuple(base)
        ctxs = [bt + tuple(int(t) for t in p) for p in paths]
        # nodes whose keys are missing (first layers, or after a reset): by depth
        need = sorted({c[:j] for c in ctxs for j in range(nb + 1, len(c)) if c[:j] not in self.node_kv}, key=len)
        while need:
            d = len(need[0])
            self._tree_rows([c for c in need if len(c) == d], nb)
            need = [c for c in need if len(c) > d]
        return self._tree_rows(ctxs, nb)

    def _tree_rows(self, ctxs: list[tuple], nb: int) -> torch.Tensor:
        c = self.cfg
        n = len(ctxs)
        nh, nkv, hd = c.n_heads, c.n_kv_heads, c.head_dim
        g = nh // nkv
        pos = torch.tensor([len(x) - 1 for x in ctxs])
        x = self.w["embed"][torch.tensor([x[-1] for x in ctxs])]
        own = [[] for _ in range(n)]
        for i in range(c.n_layers):
            p = f"l{i}."
            h = self._rms(x, self.w[p + "attn_norm"])
            q = h @ self.w[p + "wq"].T
            k = h @ self.w[p + "wk"].T
            v = h @ self.w[p + "wv"].T
            if c.qkv_bias:
                q, k, v = q + self.w[p + "bq"], k + self.w[p + "bk"], v + self.w[p + "bv"]
            q = self._rope(q.view(n, nh, hd), pos) / math.sqrt(hd)
            k = self._rope(k.view(n, nkv, hd), pos)
            v = v.view(n, nkv, hd)
            Kb, Vb = self.kv[i]
            Kb = Kb[:nb].repeat_interleave(g, dim=1)
            Vb = Vb[:nb].repeat_interleave(g, dim=1)
            sb = torch.einsum("nhd,thd->nht", q, Kb)          # every row sees the whole base
            o = torch.empty(n, nh, hd)
            for r, cx in enumerate(ctxs):
                anc = [self.node_kv[cx[:j]][i] for j in range(nb + 1, len(cx))]
                ke = torch.stack([a[0] for a in anc] + [k[r]]).repeat_interleave(g, dim=1)   # [e, nh, hd]
                ve = torch.stack([a[1] for a in anc] + [v[r]]).repeat_interleave(g, dim=1)
                se = torch.einsum("hd,ehd->he", q[r], ke)
                a = torch.softmax(torch.cat([sb[r], se], dim=-1), dim=-1)
                o[r] = torch.einsum("ht,thd->hd", a[:, :nb], Vb) + torch.einsum("he,ehd->hd", a[:, nb:], ve)
                own[r].append((k[r], v[r]))
            x = x + o.reshape(n, nh * hd) @ self.w[p + "wo"].T
            h = self._rms(x, self.w[p + "mlp_norm"])
            x = x + (torch.nn.functional.silu(h @ self.w[p + "wg"].T) * (h @ self.w[p + "wu"].T)) @ self.w[p + "wd"].T
        for r, cx in enumerate(ctxs):
            self.node_kv[cx] = own[r]
        x = self._rms(x, self.w["norm"])
        return x @ self.w["lm_head"].T


class RefModel:
    """The reference's model protocol (lm.py:109-196) over RefLlama, with the
    same optional k-gram logit bias as the device model (lm.LogitBias)."""

    def __init__(self, cfg, weights, *, params_billions=1.0, forward_latency=1.0, eos_token=None, bias=None):
        self.llama = RefLlama(cfg, weights)
        self.vocab_size = cfg.vocab_size
        self.params_billions = params_billions
        self.forward_latency = forward_latency
        self.eos_token = eos_token
        self.bias = bias

    def next_distribution(self, ctx, temperature=1.0):
        if self.eos_token is not None and ctx[-1] == self.eos_token:
            out = np.zeros(self.vocab_size)
            out[self.eos_token] = 1.0
            return out
        return self._dist(ctx, self.llama.logits_for(list(ctx)), temperature)

    def _dist(self, ctx, lg, temperature):
        if self.eos_token is not None and ctx[-1] == self.eos_token:
            out = np.zeros(self.vocab_size)
            out[self.eos_token] = 1.0
            return out
        lg = lg.double()
        if self.bias is not None and self.bias.sharpness != 0.0:
            from oracle.card_oracle import kgram_uniforms_np

            tail = [int(t) for t in ctx][-self.bias.order:]
            u = kgram_uniforms_np(self.bias.seed, tail, self.vocab_size).astype(np.float32)
            if self.bias.mix_weight:
                u = u + np.float32(self.bias.mix_weight) * kgram_uniforms_np(
                    self.bias.mix_seed, tail, self.vocab_size).astype(np.float32)
            lg = (lg.float() + torch.from_numpy(np.float32(self.bias.sharpness) * u)).double()
        if temperature == 0.0:
            out = np.zeros(self.vocab_size)
            out[int(torch.argmax(lg))] = 1.0
            return out
        return torch.softmax(lg / temperature, dim=0).numpy()


class BatchedRefModel(RefModel):
    """RefModel with the batched passes a real backend makes (lm.py:155-163:
    "a real backend would batch this into a single masked pass"): a draft
    tree layer in one masked forward (`tree_distributions`) and a verify
    chain in one forward (`chain_distributions`).  card_oracle.serial_cycles
    uses them when present; same distributions up to fp32 summation order.
    Used by bench.py's CPU legs, where one-context-at-a-time fp32 forwards
    would make a CARD cycle take minutes."""

    def tree_distributions(self, base, paths, temperature=1.0):
        lg = self.llama.tree_logits(list(base), [list(p) for p in paths])
        return [self._dist(list(base) + list(p), lg[i], temperature) for i, p in enumerate(paths)]

    def chain_distributions(self, ctx, toks, temperature=1.0):
        lg = self.llama.chain_logits(list(ctx), list(toks))
        return [self._dist(list(ctx) + list(toks[:i]), lg[i], temperature) for i in range(len(toks) + 1)]
