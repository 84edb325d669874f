"""Engine path for host-table models (``ScriptedModel`` or any user model
that only implements ``next_distribution``): the distributions are the
user's host data, so they are uploaded per step; the candidate tree,
verification and commit still run on the device through the drop-in
TreeCache / verify APIs.  Mirrors engine.py:149-317 / 392-423."""

from __future__ import annotations

import numpy as np

from .cache import CacheConfig, TreeCache
from .errors import FrontierFull
from .metrics import finalize


def _trace_cls():
    from .engine import RunResult, StepTrace

    return RunResult, StepTrace


def run_host_models(draft, target, prompt, config):
    from .engine import _check_pair, _check_prompt
    from .verify import argmax_token, sample_index, verify_greedy, verify_sampling

    RunResult, StepTrace = _trace_cls()
    _check_pair(draft, target)
    prompt = _check_prompt(prompt, target.vocab.size)
    cfg = config
    t_score = cfg.temperature if cfg.temperature > 0.0 else 1.0
    sampling = cfg.temperature > 0.0
    rng = np.random.default_rng(cfg.seed)
    eos = target.eos_token
    cache = TreeCache(prompt[-1], CacheConfig(cfg.K, cfg.k, cfg.max_depth), eos_token=eos)
    out, trace = [], []
    st = {"base": list(prompt), "done": False, "origin_tokens": None}

    def committed():
        return prompt + out

    def emit(t, hit, cl, al, ln, ev):
        trace.append(StepTrace(len(trace), t, hit, cl, al, ln, cache.alive_below_root(), ev))

    def draft_step():
        snap = cache._snapshot()
        if snap["frontier"]:
            anchor = 0 if not cfg.correction_enabled else snap["root"]
            dists = []
            for h in snap["frontier"]:
                rev, cur = [], h
                while cur != anchor:
                    rev.append(snap["token"][cur])
                    cur = snap["parent"][cur]
                dists.append(draft.next_distribution(st["base"] + rev[::-1], t_score))
        else:
            dists = [draft.next_distribution(committed(), t_score)]
        try:
            new = cache.expand_layer(np.vstack(dists))
        except FrontierFull:
            return 0
        return len(new)

    def target_step():
        res = cache.query(cfg.query_depth)
        if not res.hit:
            d = target.next_distribution(committed(), t_score)
            tok = sample_index(rng, d) if sampling else argmax_token(d)
            return False, 0, (), tok
        toks = list(res.tokens)
        ctx = committed()
        dists = [target.next_distribution(ctx + toks[:i], t_score) for i in range(len(toks) + 1)]
        o = verify_sampling(dists, [1.0] * len(toks), toks, rng) if sampling else verify_greedy(dists, toks)
        return True, len(toks), o.accepted, o.correction

    def commit(acc, corr):
        lnew = len(acc) + 1
        room = cfg.max_new_tokens - len(out)
        toks = (list(acc) + [corr])[:room]
        if eos is not None and eos in toks:
            toks = toks[: toks.index(eos) + 1]
        out.extend(toks)
        if len(toks) < lnew or len(out) >= cfg.max_new_tokens:
            st["done"] = True
        if toks and eos is not None and toks[-1] == eos:
            st["done"] = True
        return max(0, len(toks) - 1), len(toks)

    d_lat, t_lat = draft.spec.forward_latency, target.spec.forward_latency
    clock = 0.0
    for _ in range(cfg.query_depth):
        w = draft_step()
        if w == 0:
            break
        clock += d_lat
        emit(clock, False, w, 0, 0, "draft_expand")
    while not st["done"]:
        start, n_exp = clock, 0
        for _ in range(cfg.ratio):
            w = draft_step()
            if w == 0:
                break
            n_exp += 1
            emit(start + n_exp * d_lat, False, w, 0, 0, "draft_expand")
        hit, cl, acc, corr = target_step()
        clock = start + max(n_exp * d_lat, t_lat)
        a, ln = commit(acc, corr)
        emit(clock, hit, cl, a, ln, "verify" if hit else "miss_step")
        if not st["done"]:
            if cfg.correction_enabled:
                cache.correct(list(acc), corr)
                st["base"] = committed()
            elif not cache.advance_root(list(acc), corr):
                cache.reset(out[-1])
                st["base"] = committed()
            emit(clock, hit, 0, 0, 0, "correct")
    return RunResult(output=out, metrics=finalize(trace, target.spec, draft.spec), trace=trace)


def run_vanilla_host(target, prompt, config):
    from .engine import _check_prompt
    from .verify import argmax_token, sample_index

    RunResult, StepTrace = _trace_cls()
    toks = _check_prompt(prompt, target.vocab.size)
    t_score = config.temperature if config.temperature > 0.0 else 1.0
    rng = np.random.default_rng(config.seed)
    out, trace, clock = [], [], 0.0
    while len(out) < config.max_new_tokens:
        d = target.next_distribution(toks + out, t_score)
        tok = sample_index(rng, d) if config.temperature > 0.0 else argmax_token(d)
        out.append(tok)
        clock += target.spec.forward_latency
        trace.append(StepTrace(len(trace), clock, False, 0, 0, 1, 0, "miss_step"))
        if target.eos_token is not None and tok == target.eos_token:
            break
    return RunResult(output=out, metrics=finalize(trace, target.spec), trace=trace)
