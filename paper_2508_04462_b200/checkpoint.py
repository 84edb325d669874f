"""safetensors checkpoints for the transformer draft/target.

The format is an 8-byte little-endian header length, a JSON header mapping
tensor names to ``{"dtype", "shape", "data_offsets"}`` and the raw
row-major bytes.  Tensors are memory-mapped and converted to the canonical
weight dict of ``llama.init_weights`` (HF ``LlamaForCausalLM`` /
``Qwen2ForCausalLM`` names), so a loaded model goes through the same
``pack_weights`` as a random-init one.  A directory is read through its
``model.safetensors.index.json`` weight map (sharded checkpoints) or its
single ``model.safetensors``.  ``save_llama_safetensors`` writes the same
layout (tests, and converting random-init weights for other tools).
"""

from __future__ import annotations

import json
import mmap
import os
import struct

import numpy as np
import torch

from .errors import ConfigError

_DT = {"F32": (torch.float32, 4), "F16": (torch.float16, 2), "BF16": (torch.bfloat16, 2)}
_DT_NAME = {v[0]: k for k, v in _DT.items()}


def _hf_names(cfg) -> dict:
    """canonical name -> HF tensor name."""
    m = {"embed": "model.embed_tokens.weight", "norm": "model.norm.weight"}
    if not cfg.tie_embeddings:
        m["lm_head"] = "lm_head.weight"
    for i in range(cfg.n_layers):
        p, h = f"l{i}.", f"model.layers.{i}."
        for a, b in (("wq", "self_attn.q_proj.weight"), ("wk", "self_attn.k_proj.weight"),
                     ("wv", "self_attn.v_proj.weight"), ("wo", "self_attn.o_proj.weight"),
                     ("wg", "mlp.gate_proj.weight"), ("wu", "mlp.up_proj.weight"), ("wd", "mlp.down_proj.weight"),
                     ("attn_norm", "input_layernorm.weight"), ("mlp_norm", "post_attention_layernorm.weight")):
            m[p + a] = h + b
        if cfg.qkv_bias:
            for a, b in (("bq", "self_attn.q_proj.bias"), ("bk", "self_attn.k_proj.bias"),
                         ("bv", "self_attn.v_proj.bias")):
                m[p + a] = h + b
    return m


class _File:
    def __init__(self, path: str):
        try:
            self.fh = open(path, "rb")
        except OSError as exc:
            raise ConfigError(f"{path}: {exc.strerror or exc}") from None
        head = self.fh.read(8)
        if len(head) != 8:
            raise ConfigError(f"{path}: not a safetensors file")
        (n,) = struct.unpack("<Q", head)
        try:
            self.header = json.loads(self.fh.read(n))
        except (ValueError, UnicodeDecodeError) as exc:
            raise ConfigError(f"{path}: bad safetensors header ({exc})") from None
        self.base = 8 + n
        self.mm = mmap.mmap(self.fh.fileno(), 0, access=mmap.ACCESS_READ)
        self.path = path

    def tensor(self, name: str) -> torch.Tensor:
        meta = self.header[name]
        if meta["dtype"] not in _DT:
            raise ConfigError(f"{self.path}: tensor {name} has unsupported dtype {meta['dtype']}")
        dt, size = _DT[meta["dtype"]]
        a, b = meta["data_offsets"]
        count = int(np.prod(meta["shape"])) if meta["shape"] else 1
        if b - a != count * size:
            raise ConfigError(f"{self.path}: tensor {name} byte range does not match its shape")
        raw = np.frombuffer(self.mm, dtype=np.uint8, count=b - a, offset=self.base + a)
        return torch.from_numpy(raw.copy()).view(dt).reshape(meta["shape"])


def _open_all(path: str) -> dict:
    """HF tensor name -> _File holding it."""
    if os.path.isdir(path):
        index = os.path.join(path, "model.safetensors.index.json")
        if os.path.exists(index):
            with open(index, encoding="utf-8") as fh:
                wmap = json.load(fh)["weight_map"]
            files = {f: _File(os.path.join(path, f)) for f in sorted(set(wmap.values()))}
            return {name: files[f] for name, f in wmap.items()}
        path = os.path.join(path, "model.safetensors")
    f = _File(path)
    return {name: f for name in f.header if name != "__metadata__"}


def load_llama_safetensors(path: str, cfg) -> dict:
    """Canonical fp32/bf16 weight dict (llama.init_weights layout) of cfg."""
    where = _open_all(path)
    out = {}
    H, hd = cfg.hidden, cfg.head_dim
    shapes = {"embed": (cfg.vocab_size, H), "lm_head": (cfg.vocab_size, H), "norm": (H,)}
    for i in range(cfg.n_layers):
        p = f"l{i}."
        shapes.update({p + "wq": (cfg.n_heads * hd, H), p + "wk": (cfg.n_kv_heads * hd, H),
                       p + "wv": (cfg.n_kv_heads * hd, H), p + "wo": (H, cfg.n_heads * hd),
                       p + "wg": (cfg.ffn, H), p + "wu": (cfg.ffn, H), p + "wd": (H, cfg.ffn),
                       p + "attn_norm": (H,), p + "mlp_norm": (H,), p + "bq": (cfg.n_heads * hd,),
                       p + "bk": (cfg.n_kv_heads * hd,), p + "bv": (cfg.n_kv_heads * hd,)})
    for canon, hf in _hf_names(cfg).items():
        if hf not in where:
            raise ConfigError(f"{path}: checkpoint has no tensor {hf}")
        t = where[hf].tensor(hf)
        if tuple(t.shape) != shapes[canon]:
            raise ConfigError(f"{path}: {hf} has shape {tuple(t.shape)}, the config needs {shapes[canon]}")
        out[canon] = t if t.dtype == torch.bfloat16 else t.float()
    out["lm_head"] = out["embed"] if cfg.tie_embeddings else out["lm_head"]
    return out


def save_llama_safetensors(path: str, cfg, weights: dict) -> None:
    """Write canonical weights under HF names (one file)."""
    names = _hf_names(cfg)
    header, blobs, off = {}, [], 0
    for canon, hf in names.items():
        t = weights[canon].detach().cpu().contiguous()
        if t.dtype not in _DT_NAME:
            t = t.float()
        b = t.view(torch.uint8).numpy().tobytes() if t.dim() else t.reshape(1).view(torch.uint8).numpy().tobytes()
        header[hf] = {"dtype": _DT_NAME[t.dtype], "shape": list(t.shape), "data_offsets": [off, off + len(b)]}
        blobs.append(b)
        off += len(b)
    js = json.dumps(header, separators=(",", ":")).encode()
    js += b" " * ((8 - len(js) % 8) % 8)
    with open(path, "wb") as fh:
        fh.write(struct.pack("<Q", len(js)))
        fh.write(js)
        for b in blobs:
            fh.write(b)
