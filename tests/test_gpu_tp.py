"""Device tensor-parallel target (BASELINE configs[3] path).
The box has one GPU, so the ranks are processes sharing cuda:0 with a gloo
group (all-reduce on CUDA tensors); on a multi-GPU node the same code runs
one rank per GPU over NCCL.  World 2 (even) and 3 (uneven: kv heads 2/1/1,
vocabulary tiles 2/2/1): every rank's gathered logits match the unsharded
device model, and greedy CARD with the sharded target equals greedy AR of
the sharded target on every rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _cfg():
    from paper_2508_04462_b200.llama import LlamaConfig

    return LlamaConfig(640, 512, 2, 8, 4, 128, 1536, 500000.0, 1e-5, False, False, None)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2508_04462_b200 as card
    from paper_2508_04462_b200.engine import forward_context_logits
    from paper_2508_04462_b200.llama import PRESETS, init_weights
    from paper_2508_04462_b200.tp import TPComm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = _cfg()
        w = init_weights(cfg, seed=3)
        bias = card.LogitBias(seed=11, order=2, sharpness=4000.0)
        target = card.LlamaModel(cfg, dtype="bf16", weights=w, tp=TPComm(), bias=bias,
                                 spec=card.ModelSpec(8.0, 7.0))
        ctx = [int(x) for x in np.random.default_rng(4).integers(0, cfg.vocab_size, 150)]
        lg = forward_context_logits(target, ctx).cpu()
        dcfg = PRESETS["small-draft"]
        dcfg = type(dcfg)(**{**dcfg.to_dict(), "vocab_size": cfg.vocab_size})
        draft = card.LlamaModel(dcfg, dtype="bf16", weights=init_weights(dcfg, 1), bias=bias,
                                spec=card.ModelSpec(1.0, 1.0))
        prompt = ctx[:40]
        ecfg = card.EngineConfig(K=16, k=3, ratio=5, max_new_tokens=64)
        res = card.run_speculative(draft, target, prompt, ecfg)
        van = card.run_vanilla(target, prompt, ecfg)
        q.put((rank, lg, res.output, van.output, res.metrics.mean_acceptance_length))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_tp_target_on_device(world):
    import paper_2508_04462_b200 as card
    from paper_2508_04462_b200.engine import forward_context_logits
    from paper_2508_04462_b200.llama import init_weights

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        r, *rest = q.get(timeout=600)
        got[r] = rest
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = _cfg()
    full = card.LlamaModel(cfg, dtype="bf16", weights=init_weights(cfg, seed=3))
    ctx_toks = [int(x) for x in np.random.default_rng(4).integers(0, cfg.vocab_size, 150)]
    want = forward_context_logits(full, ctx_toks).cpu()
    for r in range(world):
        lg, out, van, acc = got[r]
        rel = float((lg - want).norm() / want.norm())
        assert rel < 1e-2, (r, rel)
        assert torch.equal(lg, got[0][0])         # identical on every rank
        assert out == van and out == got[0][1]    # lossless, and the ranks agree
        assert acc > 1.0
