"""Body of __graft_entry__.smoke(): one tiny CARD decode on cuda:0, checked
against the CPU oracle (test infrastructure: the oracle is the checker).

1. Device candidate tree vs the oracle's SoA restatement (cache.py:224-251).
2. Greedy CARD decode of a tiny fp32 Llama pair through the stepwise and the
   CUDA-graph drivers vs the oracle engine (engine.py:290-317) driving the
   CPU transformer with the same weights: identical tokens.
3. The same decode equals target-only autoregressive decoding (lossless).
"""


def run_smoke():
    import numpy as np
    import torch

    import paper_2508_04462_b200 as card
    from oracle import card_oracle as O
    from oracle.llama_ref import RefModel
    from paper_2508_04462_b200._device import require_cuda
    from paper_2508_04462_b200.llama import PRESETS, init_weights
    from paper_2508_04462_b200.lm import LogitBias

    require_cuda()
    # 1. cache
    cache = card.TreeCache(0, card.CacheConfig(K=4, k=2, max_depth=3))
    twin = O.SoATree(0, 4, 2, 3, log_fn=O.cr_log)
    d = np.array([[0.5, 0.3, 0.2]])
    cache.expand_layer(d)
    twin.expand(d)
    assert cache.frontier == twin.frontier, (cache.frontier, twin.frontier)

    # 2. tiny transformer pair, greedy CARD vs the oracle engine
    ct, cd = PRESETS["tiny-target"], PRESETS["tiny-draft"]
    wt, wd = init_weights(ct, 2), init_weights(cd, 1)
    bias = LogitBias(seed=11, order=2, sharpness=20.0, mix_seed=131, mix_weight=0.05)
    t = card.LlamaModel(ct, dtype="fp32", weights=wt, spec=card.ModelSpec(8.0, 7.0), bias=bias)
    dm = card.LlamaModel(cd, dtype="fp32", weights=wd, spec=card.ModelSpec(1.0, 1.0), bias=bias)
    prompt = [int(x) for x in np.random.default_rng(9).integers(0, ct.vocab_size, 16)]
    kw = dict(K=6, k=2, ratio=3, max_new_tokens=24)
    cfg = card.EngineConfig(**kw)
    step = card.run_speculative(dm, t, prompt, cfg, use_graphs=False)
    graph = card.run_speculative(dm, t, prompt, cfg, use_graphs=True)
    rd = RefModel(cd, wd, forward_latency=1.0, bias=bias)
    rt = RefModel(ct, wt, forward_latency=7.0, params_billions=8.0, bias=bias)
    want, _ = O.run_serial(rd, rt, prompt, **kw)
    assert step.output == want, (step.output, want)
    assert graph.output == want, (graph.output, want)
    # 3. lossless vs autoregressive decoding on the device
    van = card.run_vanilla(t, prompt, cfg)
    assert van.output == want, (van.output, want)
    torch.cuda.synchronize()
    print(f"smoke ok: {len(want)} tokens, mean acceptance {step.metrics.mean_acceptance_length:.3f}, "
          f"graph-mode kernel launches {graph.wall.get('gpu_launches')}")
