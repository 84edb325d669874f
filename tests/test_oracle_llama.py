"""Pin the CPU transformer oracle (oracle/llama_ref.py) against HF
transformers' LlamaForCausalLM on identical random-init weights.  CPU only."""

import pytest
import torch

from oracle.llama_ref import RefLlama


def _cfgs():
    from paper_2508_04462_b200.llama import LlamaConfig

    scaled = dict(factor=8.0, low_freq_factor=1.0, high_freq_factor=4.0, original_max_position_embeddings=64)
    return [LlamaConfig(96, 64, 2, 4, 2, 16, 128, 10000.0, 1e-5, False, False, None),
            LlamaConfig(96, 64, 2, 4, 1, 16, 128, 500000.0, 1e-5, True, False, scaled)]


def _hf_model(cfg, w):
    transformers = pytest.importorskip("transformers")
    kw = dict(vocab_size=cfg.vocab_size, hidden_size=cfg.hidden, intermediate_size=cfg.ffn,
              num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_heads, num_key_value_heads=cfg.n_kv_heads,
              head_dim=cfg.head_dim, rms_norm_eps=cfg.rms_eps, tie_word_embeddings=cfg.tie_embeddings,
              max_position_embeddings=512)
    rp = {"rope_type": "default", "rope_theta": cfg.rope_theta}
    if cfg.rope_scaling:
        rp = {"rope_type": "llama3", "rope_theta": cfg.rope_theta, **cfg.rope_scaling}
    try:
        hc = transformers.LlamaConfig(**kw, rope_parameters=rp)
    except TypeError:
        hc = transformers.LlamaConfig(**kw, rope_theta=cfg.rope_theta, rope_scaling=cfg.rope_scaling)
    m = transformers.LlamaForCausalLM(hc).eval()
    sd = {"model.embed_tokens.weight": w["embed"], "model.norm.weight": w["norm"], "lm_head.weight": w["lm_head"]}
    for i in range(cfg.n_layers):
        p, q = f"l{i}.", f"model.layers.{i}."
        sd[q + "self_attn.q_proj.weight"] = w[p + "wq"]
        sd[q + "self_attn.k_proj.weight"] = w[p + "wk"]
        sd[q + "self_attn.v_proj.weight"] = w[p + "wv"]
        sd[q + "self_attn.o_proj.weight"] = w[p + "wo"]
        sd[q + "mlp.gate_proj.weight"] = w[p + "wg"]
        sd[q + "mlp.up_proj.weight"] = w[p + "wu"]
        sd[q + "mlp.down_proj.weight"] = w[p + "wd"]
        sd[q + "input_layernorm.weight"] = w[p + "attn_norm"]
        sd[q + "post_attention_layernorm.weight"] = w[p + "mlp_norm"]
    m.load_state_dict(sd, strict=False)
    return m


@pytest.mark.parametrize("which", [0, 1])
def test_ref_llama_matches_hf(which):
    from paper_2508_04462_b200.llama import init_weights

    cfg = _cfgs()[which]
    w = init_weights(cfg, seed=7)
    w = {k: (v * 20 if k[0] == "l" and k[1].isdigit() and "norm" not in k else v) for k, v in w.items()}
    ref = RefLlama(cfg, w)
    toks = torch.randint(0, cfg.vocab_size, (1, 150), generator=torch.Generator().manual_seed(1))
    with torch.no_grad():
        hf = _hf_model(cfg, w)(toks).logits[0]
        ours = ref.full_logits(toks[0].tolist())
    assert torch.allclose(ours, hf, rtol=1e-4, atol=1e-4), (ours - hf).abs().max()


def test_ref_llama_incremental_equals_full():
    from paper_2508_04462_b200.llama import init_weights

    cfg = _cfgs()[0]
    w = init_weights(cfg, seed=3)
    ref = RefLlama(cfg, w)
    toks = list(range(5, 45))
    full = ref.full_logits(toks)
    inc = RefLlama(cfg, w)
    for n in (10, 25, 40):
        assert torch.allclose(inc.logits_for(toks[:n]), full[n - 1], atol=1e-5)
    branch = toks[:20] + [7, 8]
    assert torch.allclose(inc.logits_for(branch), RefLlama(cfg, w).full_logits(branch)[-1], atol=1e-5)


def test_safetensors_checkpoint_round_trip_and_hf(tmp_path):
    """checkpoint.load_llama_safetensors reads what HF save_pretrained writes
    (HF names, tied and untied heads) and what save_llama_safetensors writes,
    and the loaded weights give the oracle the same logits."""
    from paper_2508_04462_b200.checkpoint import load_llama_safetensors, save_llama_safetensors
    from paper_2508_04462_b200.errors import ConfigError
    from paper_2508_04462_b200.llama import init_weights

    for which in (0, 1):
        cfg = _cfgs()[which]
        w = init_weights(cfg, seed=11 + which)
        p = tmp_path / f"m{which}.safetensors"
        save_llama_safetensors(str(p), cfg, w)
        got = load_llama_safetensors(str(p), cfg)
        assert set(got) == set(w)
        assert all(torch.equal(got[k], w[k]) for k in w)
        d = tmp_path / f"hf{which}"
        _hf_model(cfg, w).save_pretrained(str(d), safe_serialization=True)
        hf = load_llama_safetensors(str(d), cfg)
        toks = list(range(3, 40))
        assert torch.equal(RefLlama(cfg, hf).full_logits(toks), RefLlama(cfg, w).full_logits(toks))
    bad = tmp_path / "bad.safetensors"
    bad.write_bytes(b"\x01\x00")
    with pytest.raises(ConfigError):
        load_llama_safetensors(str(bad), _cfgs()[0])


def test_batched_passes_equal_per_context():
    """The batched CPU passes bench.py's CPU legs use (one masked pass per
    draft tree layer, one pass per verify chain) give the per-context
    distributions, and the oracle CARD loop driven by them emits the same
    tokens and trace as the per-context protocol (lm.py:155-163)."""
    import numpy as np

    from oracle import card_oracle as O
    from oracle.llama_ref import BatchedRefModel, RefModel
    from paper_2508_04462_b200.llama import PRESETS, init_weights
    from paper_2508_04462_b200.lm import LogitBias

    cfg = _cfgs()[1]
    w = init_weights(cfg, seed=5)
    ref, bat = RefLlama(cfg, w), RefLlama(cfg, w)
    base = list(range(3, 40))
    paths = [[5], [6], [5, 9], [5, 10], [6, 11, 12], [5, 9, 13, 14]]
    got = bat.tree_logits(base, paths)
    for i, p in enumerate(paths):
        assert torch.allclose(got[i], ref.logits_for(base + p), atol=2e-5), i
    got = bat.tree_logits(base + [5], [[9, 13], [10, 2]])   # base grew: memo entries reused / pruned
    assert torch.allclose(got[0], ref.logits_for(base + [5, 9, 13]), atol=2e-5)
    assert torch.allclose(got[1], ref.logits_for(base + [5, 10, 2]), atol=2e-5)
    ch = bat.chain_logits(base, [4, 8, 1])
    for i in range(4):
        assert torch.allclose(ch[i], ref.logits_for(base + [4, 8, 1][:i]), atol=2e-5)

    cd, ct = PRESETS["tiny-draft"], PRESETS["tiny-target"]
    wd, wt = init_weights(cd, seed=1), init_weights(ct, seed=2)
    bias = LogitBias(seed=11, order=2, sharpness=3e3, mix_seed=131, mix_weight=0.5)
    prompt = [int(x) for x in np.random.default_rng(4).integers(0, ct.vocab_size, 16)]
    cfg_run = dict(K=12, k=3, ratio=3, max_new_tokens=40)
    runs = []
    for M in (RefModel, BatchedRefModel):
        runs.append(O.run_serial(M(cd, wd, forward_latency=1.0, bias=bias),
                                 M(ct, wt, forward_latency=7.0, bias=bias), prompt, **cfg_run))
    assert runs[0][0] == runs[1][0]
    assert [(e.event, e.hit, e.candidate_len, e.accepted_len) for e in runs[0][1]] == \
           [(e.event, e.hit, e.candidate_len, e.accepted_len) for e in runs[1][1]]
    assert any(e.accepted_len > 0 for e in runs[0][1])
