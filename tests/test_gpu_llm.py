"""GPU numerics of the transformer path: the tcgen05/TMA GEMM and GEMV
against torch, the fp32 forward against the CPU oracle (1e-4), the bf16
forward (1e-2 relative), and losslessness of the CARD loop on transformer
pairs (greedy output == autoregressive output)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def card():
    import paper_2508_04462_b200 as card
    from paper_2508_04462_b200._device import require_cuda

    require_cuda()
    return card


@pytest.mark.parametrize("M", [1, 2, 5, 8, 16, 37, 100, 128])
@pytest.mark.parametrize("NK", [(256, 512), (1024, 4096), (384, 1536)])
@pytest.mark.parametrize("epi", [0, 1, 3])
@pytest.mark.parametrize("layout", ["rowmajor", "tiled"])
def test_linear_bf16_vs_torch(card, M, NK, epi, layout):
    from paper_2508_04462_b200.llama import _Linear, tile_sw128

    N, K = NK
    g = torch.Generator(device="cuda").manual_seed(M * 131 + N + epi)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    mpad = ((M + 15) // 16) * 16
    X = torch.zeros(mpad, K, device="cuda", dtype=torch.bfloat16)
    X[:M] = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    ref = X[:M].float() @ W.float().T
    dM = torch.tensor([M], dtype=torch.int32, device="cuda")
    if layout == "tiled":
        W = tile_sw128(W)
    if epi == 3:
        out = torch.zeros(mpad, N // 2, device="cuda", dtype=torch.bfloat16)
        lin = _Linear(W, X, M, 3, out, N // 2)
        lin.run(dM)
        torch.cuda.synchronize()
        t = ref.view(M, N // 32, 2, 16)   # interleave_gate_up: 16 gate rows, 16 up rows
        want = (torch.nn.functional.silu(t[:, :, 0]) * t[:, :, 1]).reshape(M, N // 2)
        got = out[:M].float()
        assert torch.allclose(got, want, rtol=2e-2, atol=2e-2), (got - want).abs().max()
        return
    out = torch.randn(mpad, N, device="cuda", generator=g) if epi == 1 else torch.zeros(mpad, N, device="cuda")
    before = out.clone()
    lin = _Linear(W, X, M, epi, out, N)
    lin.run(dM)
    torch.cuda.synchronize()
    want = ref + (before[:M] if epi == 1 else 0)
    assert torch.allclose(out[:M], want, rtol=1e-3, atol=1e-3), ((out[:M] - want).abs().max(), lin.info)
    assert torch.equal(out[M:], before[M:]), "rows beyond M must not be written"


def test_linear_deterministic_and_graph_replay(card):
    from paper_2508_04462_b200.llama import _Linear

    W = (torch.randn(4096, 4096, device="cuda") * 0.02).to(torch.bfloat16)
    X = torch.randn(16, 4096, device="cuda").to(torch.bfloat16)
    out = torch.zeros(16, 4096, device="cuda")
    dM = torch.tensor([8], dtype=torch.int32, device="cuda")
    lin = _Linear(W, X, 8, 0, out, 4096)
    assert lin.info["splits"] >= 1
    lin.run(dM)
    first = out.clone()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        lin.run(dM)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, first)   # split-K fixup is order-deterministic


def _tiny_pair(card, dtype, preset_t="tiny-target", preset_d="tiny-draft", bias=None):
    from paper_2508_04462_b200.llama import PRESETS, init_weights

    ct, cd = PRESETS[preset_t], PRESETS[preset_d]
    wt, wd = init_weights(ct, 2), init_weights(cd, 1)
    spec_t = card.ModelSpec(8.0, 7.0)
    spec_d = card.ModelSpec(1.0, 1.0)
    t = card.LlamaModel(ct, dtype=dtype, weights=wt, spec=spec_t, bias=bias)
    d = card.LlamaModel(cd, dtype=dtype, weights=wd, spec=spec_d, bias=bias)
    return d, t, wd, wt, cd, ct


def test_fp32_forward_matches_cpu_oracle(card):
    from oracle.llama_ref import RefLlama
    from paper_2508_04462_b200.engine import forward_context_logits

    d, t, wd, wt, cd, ct = _tiny_pair(card, "fp32")
    rng = np.random.default_rng(0)
    ctx = [int(x) for x in rng.integers(0, ct.vocab_size, 200)]
    got = forward_context_logits(t, ctx).cpu()
    want = RefLlama(ct, wt).full_logits(ctx)[-1]
    assert torch.allclose(got, want, rtol=1e-4, atol=1e-4), (got - want).abs().max()


def test_bf16_forward_close_to_cpu_oracle(card):
    from oracle.llama_ref import RefLlama
    from paper_2508_04462_b200.engine import forward_context_logits
    from paper_2508_04462_b200.llama import PRESETS, init_weights

    ct = PRESETS["small-target"]
    w = init_weights(ct, 4)
    wb = {k: v.to(torch.bfloat16).float() for k, v in w.items()}   # oracle sees the same rounded weights
    m = card.LlamaModel(ct, dtype="bf16", weights=w)
    ctx = [int(x) for x in np.random.default_rng(1).integers(0, ct.vocab_size, 300)]
    got = forward_context_logits(m, ctx).cpu()
    want = RefLlama(ct, wb).full_logits(ctx)[-1]
    rel = (got - want).norm() / want.norm()
    assert rel < 1e-2, rel


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_card_greedy_is_lossless_on_transformers(card, dtype):
    from paper_2508_04462_b200.lm import LogitBias

    preset = ("tiny-target", "tiny-draft") if dtype == "fp32" else ("small-target", "small-draft")
    bias = LogitBias(seed=11, order=2, sharpness=30.0, mix_seed=131, mix_weight=0.05)
    d, t, *_ = _tiny_pair(card, dtype, *preset, bias=bias)
    prompt = [int(x) for x in np.random.default_rng(3).integers(0, t.vocab.size, 40)]
    cfg = card.EngineConfig(K=12, k=3, ratio=4, max_new_tokens=96)
    van = card.run_vanilla(t, prompt, cfg)
    step = card.run_speculative(d, t, prompt, cfg, use_graphs=False)
    graph = card.run_speculative(d, t, prompt, cfg, use_graphs=True)
    assert step.output == van.output
    assert graph.output == van.output
    strip = lambda tr: [(e.event, e.hit, e.candidate_len, e.accepted_len, e.lnew, e.sim_time) for e in tr]  # noqa
    assert strip(graph.trace) == strip(step.trace)
    assert step.metrics.mean_acceptance_length > 1.0


@pytest.mark.parametrize("case", [
    dict(seed=9, sharp=20.0, mix=0.05, cfg=dict(K=6, k=2, ratio=3, max_new_tokens=40)),
    dict(seed=3, sharp=40.0, mix=0.0, cfg=dict(K=10, k=3, ratio=4, max_new_tokens=48)),
    dict(seed=5, sharp=10.0, mix=0.2, cfg=dict(K=4, k=1, ratio=2, max_new_tokens=32)),
    dict(seed=7, sharp=30.0, mix=0.05, cfg=dict(K=8, k=3, ratio=5, max_new_tokens=40, correction_enabled=False)),
    # small K, long decode: the reference's 75 %-dead rule never fires (the
    # committed chain stays alive), so the fixed device arena compacts under
    # capacity pressure; the order-preserving compaction changes no decision
    dict(seed=4, sharp=40.0, mix=0.0, cfg=dict(K=2, k=2, ratio=6, max_new_tokens=400)),
])
def test_fp32_card_matches_oracle_engine(card, case):
    """Greedy fp32 runs: the device engine and the oracle engine (the
    reference schedule, engine.py:290-317, driving the CPU transformer) emit
    identical tokens and an identical trace — hits, candidate lengths,
    accepted-prefix lengths and committed counts per step, and the tree size
    after every step (cache.py:174-184)."""
    from oracle import card_oracle as O
    from oracle.llama_ref import RefModel
    from paper_2508_04462_b200.lm import LogitBias

    bias = LogitBias(seed=11, order=2, sharpness=case["sharp"], mix_seed=131, mix_weight=case["mix"])
    d, t, wd, wt, cd, ct = _tiny_pair(card, "fp32", bias=bias)
    prompt = [int(x) for x in np.random.default_rng(case["seed"]).integers(0, ct.vocab_size, 16)]
    cfg = case["cfg"]
    res = card.run_speculative(d, t, prompt, card.EngineConfig(**cfg), use_graphs=False)
    rd = RefModel(cd, wd, forward_latency=1.0, bias=bias)
    rt = RefModel(ct, wt, forward_latency=7.0, params_billions=8.0, bias=bias)
    out, trace = O.run_serial(rd, rt, prompt, **cfg)
    assert res.output == out
    strip = lambda tr: [(e.event, e.hit, e.candidate_len, e.accepted_len, e.lnew, e.cache_alive_nodes)  # noqa: E731
                        for e in tr]
    assert strip(res.trace) == strip(trace)


def test_card_greedy_lossless_high_acceptance_bf16(card):
    """bf16 CARD at high acceptance (long verify chains, M up to r+1 rows)
    emits exactly the greedy AR tokens: the verify forward must compute each
    row bit-identically to a 1-row forward (no M-dependent reduction order)."""
    from paper_2508_04462_b200.lm import LogitBias

    bias = LogitBias(seed=11, order=2, sharpness=4000.0, mix_seed=131, mix_weight=0.0)
    d, t, *_ = _tiny_pair(card, "bf16", "small-target", "small-draft", bias=bias)
    prompt = [int(x) for x in np.random.default_rng(5).integers(0, t.vocab.size, 64)]
    cfg = card.EngineConfig(K=24, k=3, ratio=7, max_new_tokens=256)
    van = card.run_vanilla(t, prompt, cfg)
    res = card.run_speculative(d, t, prompt, cfg, use_graphs=True)
    assert res.metrics.mean_acceptance_length > 2.5, res.metrics.mean_acceptance_length
    assert res.output == van.output


@pytest.mark.parametrize("exchange", ["events", "mailbox"])
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_concurrent_mode_is_lossless(card, dtype, exchange):
    """mode="concurrent" (engine.py:320-389): draft and target on two streams,
    exchanging queries and corrections through stream events + a device
    hand-off, or through the device mailboxes (csrc/card_mailbox.cu: the
    target's verify graph blocks on the query box, each draft step polls
    the commit box); greedy tokens equal autoregressive decoding, also for a
    second request on the same session (the mailboxes are reset)."""
    from paper_2508_04462_b200.lm import LogitBias

    preset = ("tiny-target", "tiny-draft") if dtype == "fp32" else ("small-target", "small-draft")
    sharp = 30.0 if dtype == "fp32" else 4000.0
    bias = LogitBias(seed=11, order=2, sharpness=sharp, mix_seed=131, mix_weight=0.0)
    d, t, *_ = _tiny_pair(card, dtype, *preset, bias=bias)
    if exchange == "mailbox":
        # one GPU: the verify graph's mailbox wait and the draft's cooperative
        # persistent forward cannot share the SMs (the driver refuses the mix)
        d.persistent = False
    prompt = [int(x) for x in np.random.default_rng(7).integers(0, t.vocab.size, 48)]
    cfg = card.EngineConfig(K=16, k=3, ratio=5, max_new_tokens=160, mode="concurrent")
    van = card.run_vanilla(t, prompt, cfg)
    res = card.run_speculative(d, t, prompt, cfg, use_graphs=True, exchange=exchange)
    assert res.output == van.output
    assert res.wall["target_steps"] < len(res.output)   # more than one token per verify on average
    events = {e.event for e in res.trace}
    assert {"verify", "correct"} <= events
    prompt2 = [int(x) for x in np.random.default_rng(17).integers(0, t.vocab.size, 48)]
    again = card.run_speculative(d, t, prompt2, cfg, use_graphs=True, exchange=exchange)
    assert again.output == card.run_vanilla(t, prompt2, cfg).output


@pytest.mark.parametrize("exchange", ["events", "mailbox"])
@pytest.mark.parametrize("devices", [(0, 0), (0, 1)])
def test_concurrent_device_placement(card, devices, exchange):
    """Draft||target placement of mode="concurrent": the tree and draft state
    on the draft device, committed tokens and target state on the target
    device, each side reading the other's small buffers directly (P2P over
    NVLink on two GPUs; (0, 0) exercises the same code on one)."""
    import torch

    from paper_2508_04462_b200.llama import PRESETS, init_weights
    from paper_2508_04462_b200.lm import LogitBias

    if max(devices) >= torch.cuda.device_count():
        pytest.skip("needs two GPUs")
    if exchange == "mailbox" and devices[0] == devices[1]:
        pytest.skip("one-GPU mailbox runs are covered by test_concurrent_mode_is_lossless")
    bias = LogitBias(seed=11, order=2, sharpness=4000.0)
    ct, cd = PRESETS["small-target"], PRESETS["small-draft"]
    with torch.cuda.device(devices[1]):
        t = card.LlamaModel(ct, dtype="bf16", weights=init_weights(ct, 2), spec=card.ModelSpec(8.0, 7.0), bias=bias)
    with torch.cuda.device(devices[0]):
        d = card.LlamaModel(cd, dtype="bf16", weights=init_weights(cd, 1), spec=card.ModelSpec(1.0, 1.0), bias=bias)
    prompt = [int(x) for x in np.random.default_rng(8).integers(0, t.vocab.size, 40)]
    cfg = card.EngineConfig(K=16, k=3, ratio=5, max_new_tokens=128, mode="concurrent")
    with torch.cuda.device(devices[1]):
        van = card.run_vanilla(t, prompt, cfg)
    res = card.run_speculative(d, t, prompt, cfg, use_graphs=True, devices=devices, exchange=exchange)
    assert res.output == van.output
    assert res.wall["target_steps"] < len(res.output)


@pytest.mark.parametrize("exchange", ["events"])
def test_concurrent_sm_partitions_are_lossless(card, exchange):
    """mode="concurrent" with the GPU split into a draft and a target SM
    partition (card_green; draft_sms): graphs captured on the partition
    streams, the draft's persistent forward sized to its share; greedy
    tokens still equal autoregressive decoding."""
    from paper_2508_04462_b200.lm import LogitBias

    bias = LogitBias(seed=11, order=2, sharpness=4000.0)
    d, t, *_ = _tiny_pair(card, "bf16", "small-target", "small-draft", bias=bias)
    prompt = [int(x) for x in np.random.default_rng(9).integers(0, t.vocab.size, 48)]
    cfg = card.EngineConfig(K=16, k=3, ratio=5, max_new_tokens=96, mode="concurrent")
    res = card.run_speculative(d, t, prompt, cfg, use_graphs=True, exchange=exchange, draft_sms=48)
    assert res.output == card.run_vanilla(t, prompt, cfg).output


def test_mailbox_refused_next_to_the_persistent_draft(card):
    from paper_2508_04462_b200.errors import ConfigError
    from paper_2508_04462_b200.lm import LogitBias

    d, t, *_ = _tiny_pair(card, "bf16", "small-target", "small-draft", bias=LogitBias(seed=11, order=2,
                                                                                       sharpness=4000.0))
    prompt = [int(x) for x in np.random.default_rng(7).integers(0, t.vocab.size, 48)]
    cfg = card.EngineConfig(K=16, k=3, ratio=5, max_new_tokens=16, mode="concurrent")
    with pytest.raises(ConfigError):
        card.run_speculative(d, t, prompt, cfg, use_graphs=True, exchange="mailbox")
    with pytest.raises(ConfigError):   # nor on SM partitions of one GPU
        card.run_speculative(d, t, prompt, cfg, use_graphs=True, exchange="mailbox", draft_sms=48)


@pytest.mark.parametrize("mode", ["serial_sim", "concurrent"])
def test_eos_on_transformer_pair(card, mode):
    """An EOS-producing pair (lm.py:148-150 absorbing EOS, cache.py EOS parents
    never extended, engine.py:247-262 clipping): CARD stops exactly where
    greedy AR stops."""
    from paper_2508_04462_b200.lm import LogitBias

    bias = LogitBias(seed=11, order=2, sharpness=4000.0)
    d, t, *_ = _tiny_pair(card, "bf16", "small-target", "small-draft", bias=bias)
    prompt = [int(x) for x in np.random.default_rng(12).integers(0, t.vocab.size, 32)]
    cfg = card.EngineConfig(K=16, k=3, ratio=4, max_new_tokens=200, mode=mode)
    free = card.run_vanilla(t, prompt, cfg).output
    eos = free[len(free) // 3]                   # a token greedy decoding emits early on
    t.eos_token = d.eos_token = eos
    van = card.run_vanilla(t, prompt, cfg)
    res = card.run_speculative(d, t, prompt, cfg, use_graphs=True)
    assert van.output[-1] == eos and len(van.output) <= len(free) // 3 + 1
    assert res.output == van.output


def test_batch_of_requests_equals_single_runs(card):
    """run_speculative_batch (several requests interleaved on their own
    streams, BASELINE configs[4]): every request's tokens and trace equal a
    single run of the same prompt."""
    from paper_2508_04462_b200.lm import LogitBias

    bias = LogitBias(seed=11, order=2, sharpness=4000.0)
    d, t, *_ = _tiny_pair(card, "bf16", "small-target", "small-draft", bias=bias)
    rng = np.random.default_rng(21)
    prompts = [[int(x) for x in rng.integers(0, t.vocab.size, n)] for n in (24, 40, 33)]
    cfg = card.EngineConfig(K=16, k=3, ratio=5, max_new_tokens=96)
    batch, timing = card.run_speculative_batch(d, t, prompts, cfg)
    assert timing["requests"] == 3 and timing["tokens"] == sum(len(r.output) for r in batch)
    strip = lambda tr: [(e.event, e.hit, e.candidate_len, e.accepted_len, e.lnew) for e in tr]  # noqa: E731
    for p, got in zip(prompts, batch):
        one = card.run_speculative(d, t, p, cfg)
        assert got.output == one.output
        assert strip(got.trace) == strip(one.trace)


@pytest.mark.parametrize("mode,temperature", [("serial_sim", 0.0), ("serial_sim", 1.0), ("concurrent", 0.0)])
def test_session_reuse_equals_fresh_runs(card, mode, temperature):
    """run_speculative keeps a serving session (device buffers and the two
    captured graphs) per (pair, config, prompt length).  A request on a reused
    session emits exactly the tokens, trace and metrics of a fresh run."""
    from paper_2508_04462_b200.lm import LogitBias

    bias = LogitBias(seed=11, order=2, sharpness=4000.0)
    d, t, *_ = _tiny_pair(card, "bf16", "small-target", "small-draft", bias=bias)
    cfg = card.EngineConfig(K=16, k=3, ratio=4, max_new_tokens=96, temperature=temperature, seed=3, mode=mode)
    prompts = [[int(x) for x in np.random.default_rng(40 + i).integers(0, t.vocab.size, 32)] for i in range(3)]
    fresh = []
    for p in prompts:
        t.__dict__.pop("_card_sessions", None)
        fresh.append(card.run_speculative(d, t, p, cfg, use_graphs=True))
    t.__dict__.pop("_card_sessions", None)
    for i in [0, 1, 2, 0, 2]:
        res = card.run_speculative(d, t, prompts[i], cfg, use_graphs=True)
        assert res.output == fresh[i].output
        if mode == "concurrent":   # greedy tokens are schedule-invariant; the wall-clock trace is not
            continue
        assert [e.to_dict() for e in res.trace] == [e.to_dict() for e in fresh[i].trace]
        assert res.metrics == fresh[i].metrics
    assert len(t._card_sessions) == 1
    if temperature > 0.0:
        return
    # a changed EOS is part of the session key: the next run builds a new session
    t.eos_token = d.eos_token = fresh[0].output[5]
    res = card.run_speculative(d, t, prompts[0], cfg, use_graphs=True)
    assert len(t._card_sessions) == 2 and res.output[-1] == t.eos_token


def test_lm_head_fused_kgram_bias_is_bit_identical(card):
    """card_linear_fuse_kgram: the lm_head epilogue adds the k-gram logit bias
    with the same fp32 arithmetic as card_logit_bias applied afterwards."""
    from paper_2508_04462_b200._device import ptr, stream_ptr
    from paper_2508_04462_b200._lib import lib
    from paper_2508_04462_b200.llama import RowBlock
    from paper_2508_04462_b200.lm import LogitBias

    bias = LogitBias(seed=11, order=2, sharpness=4000.0)
    d, t, *_ = _tiny_pair(card, "bf16", "small-target", "small-draft", bias=bias)
    m = 24
    rt = d.runtime(256, 64, {m})
    assert rt.fused
    V = d.cfg.vocab_size
    rows = RowBlock(m, 16, rt.dev)
    rows.set_chain([int(x) for x in np.random.default_rng(3).integers(0, V, m)], 100, out_last_only=False)
    tail = torch.randint(0, V, (m, 2), dtype=torch.int32, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    tail[3, 0] = -1   # a short context
    rt.forward(rows, m)
    want = rt.logits[:m].clone()
    raise_for_status = card.errors.raise_for_status
    raise_for_status(lib().card_logit_bias(ptr(want), ptr(rows.n_out), m, V, ptr(tail), 2, 2, 11, 131, 0.0, 4000.0,
                                           stream_ptr()), "logit_bias")
    lm = rt.plans[m]["lm_head"]
    raise_for_status(lib().card_linear_fuse_kgram(lm.h, ptr(tail), 2, 2, 11, 131, 0.0, 4000.0), "fuse")
    rt.forward(rows, m)
    raise_for_status(lib().card_linear_fuse_kgram(lm.h, None, 0, 0, 0, 0, 0.0, 0.0), "fuse off")
    torch.cuda.synchronize()
    assert torch.equal(rt.logits[:m], want)
    rt.forward(rows, m)   # and off again
    torch.cuda.synchronize()
    assert not torch.equal(rt.logits[:m], want)


@pytest.mark.parametrize("m", [1, 24, 116])
@pytest.mark.parametrize("sharp,temp", [(0.0, 1.0), (4000.0, 1.0), (4000.0, 0.8)])
def test_fused_lm_head_topk_matches_logits_path(card, m, sharp, temp):
    """the EPI_TOPK lm_head (per vocab-tile top-4 + sum-exp records,
    card_lmhead_topk_merge) returns the tokens of the logits + top-k reader
    path, and the same log-probs up to the fp32 partial-sum order."""
    from paper_2508_04462_b200._device import ptr, stream_ptr
    from paper_2508_04462_b200._lib import lib
    from paper_2508_04462_b200.llama import RowBlock
    from paper_2508_04462_b200.lm import LogitBias

    d, t, *_ = _tiny_pair(card, "bf16", "small-target", "small-draft", bias=LogitBias(seed=11, order=2, sharpness=sharp))
    rt = d.runtime(256, 64, {m})
    V, k = d.cfg.vocab_size, 3
    rows = RowBlock(m, 16, rt.dev)
    rows.set_chain([int(x) for x in np.random.default_rng(m).integers(0, V, m)], 100, out_last_only=False)
    g = torch.Generator("cuda").manual_seed(m + 1)
    tail = torch.randint(0, V, (m, 2), dtype=torch.int32, device="cuda", generator=g)
    bias = (ptr(tail), 2, 2, 11, 131, 0.0, sharp) if sharp else (None, 0, 0, 0, 0, 0.0, 0.0)
    chk = card.errors.raise_for_status
    L = lib()
    out = [(torch.zeros((m, k), dtype=torch.int32, device="cuda"), torch.zeros((m, k), dtype=torch.float64, device="cuda"),
            torch.zeros(m, dtype=torch.int32, device="cuda")) for _ in range(2)]
    rt.forward(rows, m)
    wk = torch.zeros(L.card_lmhead_work_floats(m, k), dtype=torch.float32, device="cuda")
    chk(L.card_topk_logits(ptr(rt.logits), ptr(rows.n_out), m, V, k, 1.0 / temp, ptr(out[0][0]), ptr(out[0][1]),
                           ptr(out[0][2]), ptr(wk), *bias, stream_ptr()), "topk_logits")
    head = rt.lm_topk_head(m)
    chk(L.card_linear_fuse_kgram(head.h, *bias), "fuse_kgram")
    chk(L.card_linear_fuse_topk(head.h, V, 1.0 / temp), "fuse_topk")
    rt.forward(rows, m, topk=True)
    chk(L.card_lmhead_topk_merge(ptr(head.work), ptr(rows.n_out), m, head.n_tiles, k, V, ptr(out[1][0]),
                                 ptr(out[1][1]), ptr(out[1][2]), stream_ptr()), "merge")
    torch.cuda.synchronize()
    assert torch.equal(out[1][0], out[0][0])
    assert torch.equal(out[1][2], out[0][2])
    assert (out[1][1] - out[0][1]).abs().max().item() < 2e-5
