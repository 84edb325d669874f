"""CPU oracle for the CARD query-and-correct loop — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The shipped package
(``paper_2508_04462_b200``) must never route through it.

It restates the reference ``specache`` algorithm (read-only at
/root/reference/pkg/src/specache) operation for operation, but stores the
candidate tree the way the device does: a struct-of-arrays arena
(token / parent / layer / log_score / edge_logp / alive) plus a frontier
list, so device snapshots can be compared field by field.

Parity pin: ``tests/golden/*.json`` were produced by running the reference
itself (``oracle/make_golden.py``); ``tests/test_oracle.py`` checks this
restatement against every one of them, and against the reference's own
committed goldens (ablation.json / ksweep.json).

Citations (file:line) are into /root/reference/pkg/src/specache/.
"""

from __future__ import annotations

import decimal
import math
from dataclasses import dataclass, field

import numpy as np

_CTX = decimal.Context(prec=50)


def _D(x: float) -> decimal.Decimal:
    return _CTX.create_decimal(x)

# --------------------------------------------------------------------------
# hashed k-gram "forward" and row top-k  (_kernels_py.py:17-119)
# --------------------------------------------------------------------------

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
MIX_C1 = 0xBF58476D1CE4E5B9
MIX_C2 = 0x94D049BB133111EB
SEED_SALT = 0xD1B54A32D192ED03
INV_2_53 = 1.0 / 9007199254740992.0


def mix64(z: int) -> int:
    """splitmix64 finaliser (_kernels_py.py:27-32)."""
    z &= M64
    z = ((z ^ (z >> 30)) * MIX_C1) & M64
    z = ((z ^ (z >> 27)) * MIX_C2) & M64
    return z ^ (z >> 31)


def stream_state(seed: int, tail) -> int:
    """(_kernels_py.py:35-40)"""
    s = mix64(((seed & M64) + SEED_SALT) & M64)
    for t in tail:
        s = mix64(s ^ mix64((int(t) + 1) & M64))
    return s


def kgram_uniforms(seed: int, tail, n: int) -> list[float]:
    s = stream_state(seed, tail)
    return [(mix64((s + (i + 1) * GAMMA) & M64) >> 11) * INV_2_53 for i in range(n)]


def kgram_uniforms_np(seed: int, tail, n: int) -> np.ndarray:
    """kgram_uniforms vectorised (uint64 wrap-around arithmetic): the same
    float64 values, for vocabulary-sized rows in the CPU baselines."""
    s = np.uint64(stream_state(seed, tail))
    with np.errstate(over="ignore"):
        z = s + np.arange(1, n + 1, dtype=np.uint64) * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX_C1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX_C2)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * INV_2_53


def cr_log(x: float) -> float:
    """Correctly rounded natural log (50-digit decimal, then one rounding).
    glibc's math.log (what the reference calls) is misrounded by 1 ulp on
    ~0.04% of inputs; the device implements the correctly rounded one, so
    bit-exact device parity is checked against this twin."""
    if x == 1.0:
        return 0.0
    return float(_D(x).ln(_CTX))


def cr_exp(x: float) -> float:
    """Correctly rounded exp (see cr_log)."""
    if x < -745.2:
        return 0.0
    return float(_D(x).exp(_CTX))


def kgram_dist(seed, seed2, mix_weight, tail, vocab_size, sharpness, temperature,
               exp_fn=math.exp) -> np.ndarray:
    """(_kernels_py.py:48-102): uniforms -> optional mix -> fp64 softmax
    with a sequential sum; temperature 0 is a first-max one-hot."""
    n = vocab_size
    u = kgram_uniforms(seed, tail, n)
    if mix_weight != 0.0:
        u2 = kgram_uniforms(seed2, tail, n)
        u = [u[i] + mix_weight * u2[i] for i in range(n)]
    out = np.zeros(n, dtype=np.float64)
    if temperature == 0.0:
        best, best_v = 0, sharpness * u[0]
        for i in range(1, n):
            a = sharpness * u[i]
            if a > best_v:
                best, best_v = i, a
        out[best] = 1.0
        return out
    b = [(sharpness * x) / temperature for x in u]
    m = max(b)
    z = 0.0
    for i in range(n):
        b[i] = exp_fn(b[i] - m)
        z = z + b[i]
    for i in range(n):
        out[i] = b[i] / z
    return out


def rows_topk(dists, k: int) -> list[list[tuple[int, float]]]:
    """Per-row top-k by (p desc, token asc), p <= 0 excluded (_kernels_py.py:105-119)."""
    out = []
    for row in np.asarray(dists, dtype=np.float64):
        cand = [(float(row[t]), t) for t in range(row.shape[0]) if row[t] > 0.0]
        cand.sort(key=lambda e: (-e[0], e[1]))
        out.append([(t, p) for p, t in cand[:k]])
    return out


# --------------------------------------------------------------------------
# errors (errors.py:6-45) — the oracle raises plain types with the same names
# --------------------------------------------------------------------------

class OracleFrontierFull(Exception):
    pass


class OracleProtocolError(Exception):
    pass


class OracleInputError(Exception):
    pass


# --------------------------------------------------------------------------
# SoA candidate tree (cache.py:92-523)
# --------------------------------------------------------------------------

COMPACT_MIN_ARENA = 64          # cache.py:30
COMPACT_DEAD_FRACTION = 0.75    # cache.py:31


class SoATree:
    """Arena beam tree with the reference's exact ordering rules.

    Arena ids grow monotonically and compaction preserves order, so a
    node's children in creation order are exactly the nodes whose parent
    is it, in id order (the device relies on this; ``kids`` is only an
    index over ``parent``).
    """

    def __init__(self, root_token: int, K: int, k: int, max_depth: int, eos_token=None,
                 log_fn=math.log):
        self.K, self.k, self.max_depth, self.eos = K, k, max_depth, eos_token
        self.log_fn = log_fn
        self.epoch = 0
        self._init_root(root_token)

    # -- storage -------------------------------------------------------------
    def _init_root(self, token):                       # cache.py:111-117
        self.token = [int(token)]
        self.parent = [-1]
        self.layer = [0]
        self.score = [0.0]
        self.edge = [0.0]
        self.alive = [True]
        self.kids: list[list[int]] = [[]]   # creation-ordered child index
        self.root = 0
        self.frontier: list[int] = []
        self.dead = 0

    def _append(self, token, parent, score, edge) -> int:   # cache.py:119-131
        h = len(self.token)
        self.token.append(int(token))
        self.parent.append(parent)
        self.layer.append(self.layer[parent] + 1)
        self.score.append(score)
        self.edge.append(edge)
        self.alive.append(True)
        self.kids.append([])
        self.kids[parent].append(h)
        return h

    def children(self, h) -> list[int]:
        return self.kids[h]

    def alive_children(self, h) -> list[int]:
        return [c for c in self.children(h) if self.alive[c]]

    # -- read side -----------------------------------------------------------
    def depth_below_root(self) -> int:                 # cache.py:140-144
        if not self.frontier:
            return 0
        return self.layer[self.frontier[0]] - self.layer[self.root]

    def expansion_parents(self) -> list[int]:          # cache.py:146-149
        return list(self.frontier) if self.frontier else [self.root]

    def path_to(self, h, anchor=None) -> list[int]:    # cache.py:151-162
        anchor = self.root if anchor is None else anchor
        rev = []
        while h != anchor:
            if h < 0:
                raise OracleProtocolError("node does not descend from the anchor")
            rev.append(h)
            h = self.parent[h]
        return rev[::-1]

    def descends(self, h, anc) -> bool:                # cache.py:446-452
        while h >= 0:
            if h == anc:
                return True
            h = self.parent[h]
        return False

    def alive_below_root(self) -> int:                 # cache.py:174-184
        count, stack = 0, list(self.children(self.root))
        while stack:
            h = stack.pop()
            if not self.alive[h]:
                continue
            count += 1
            stack.extend(self.children(h))
        return count

    # -- expansion -----------------------------------------------------------
    def pool(self, dists) -> list[tuple[float, int, int, float]]:
        """(weight, token, parent_index, edge) tuples (cache.py:190-222)."""
        parents = self.expansion_parents()
        d = np.asarray(dists, dtype=np.float64)
        if d.ndim != 2 or d.shape[0] != len(parents):
            raise OracleInputError("distribution count does not match expansion parents")
        if np.isnan(d).any() or (d < 0.0).any():
            raise OracleInputError("NaN or negative")
        if np.abs(d.sum(axis=1) - 1.0).max() > 1e-9:
            raise OracleInputError("rows must sum to 1 within 1e-9")
        out = []
        for idx, (h, row) in enumerate(zip(parents, rows_topk(d, self.k))):
            if self.eos is not None and self.token[h] == self.eos:
                continue
            for tok, p in row:
                e = self.log_fn(p)
                out.append((self.score[h] + e, tok, idx, e))
        return out

    def expand(self, dists) -> list[int]:              # cache.py:224-251
        if self.depth_below_root() >= self.max_depth:
            raise OracleFrontierFull()
        parents = self.expansion_parents()
        pool = self.pool(dists)
        pool.sort(key=lambda c: (-c[0], c[1], parents[c[2]]))
        old = self.frontier
        self.frontier = [self._append(t, parents[pi], w, e) for w, t, pi, e in pool[: self.K]]
        self._prune(old)
        return list(self.frontier)

    def _prune(self, old):                             # cache.py:253-271
        keep = set()
        for h in self.frontier:
            cur = self.parent[h]
            while cur >= 0 and cur not in keep:
                keep.add(cur)
                cur = self.parent[cur]
        for h in old:
            cur = h
            while cur != self.root and cur not in keep and cur >= 0:
                if not self.alive[cur] or self.alive_children(cur):
                    break
                self.alive[cur] = False
                self.dead += 1
                cur = self.parent[cur]

    # -- query ---------------------------------------------------------------
    def query(self, depth: int):                       # cache.py:277-318
        """Returns (hit, path, tokens, edges)."""
        if not self.alive_children(self.root):
            return False, [], [], []
        d = min(depth, self.depth_below_root())
        target = self.layer[self.root] + d
        best = None
        for h in self.frontier:
            cur = h
            while self.layer[cur] > target:
                cur = self.parent[cur]
            if cur == self.root or not self.descends(cur, self.root):
                continue
            key = (-self.score[cur], self.token[cur], cur)
            if best is None or key < best:
                best = key
        assert best is not None
        path = self.path_to(best[2])
        return True, path, [self.token[h] for h in path], [self.edge[h] for h in path]

    # -- correction ----------------------------------------------------------
    def child_with(self, h, tok):                      # cache.py:337-342
        for c in self.children(h):
            if self.alive[c] and self.token[c] == tok:
                return c
        return None

    def walk(self, accepted) -> list[int]:             # cache.py:324-335
        chain, cur = [], self.root
        for t in accepted:
            nxt = self.child_with(cur, int(t))
            if nxt is None:
                raise OracleProtocolError(f"accepted token {t} not cached at depth {len(chain)}")
            chain.append(nxt)
            cur = nxt
        return chain

    def _kill(self, h):                                # cache.py:344-353
        stack = [h]
        while stack:
            x = stack.pop()
            if not self.alive[x]:
                continue
            self.alive[x] = False
            self.dead += 1
            stack.extend(self.children(x))

    def correct(self, accepted, corr) -> int:          # cache.py:355-413
        chain = self.walk(accepted)
        anchor = chain[-1] if chain else self.root
        fresh = False
        if corr is None:
            if not chain:
                raise OracleInputError("need a chain or a correction token")
            new_root = anchor
        else:
            found = self.child_with(anchor, int(corr))
            if found is None:
                new_root = self._append(corr, anchor, self.score[anchor], 0.0)
                fresh = True
            else:
                new_root = found
        path = [self.root] + chain + ([new_root] if new_root != anchor else [])
        for a, b in zip(path, path[1:]):
            for c in self.children(a):
                if c != b and self.alive[c]:
                    self._kill(c)
        old = self.frontier
        self.root = new_root
        if fresh:
            surv = []
        else:
            surv = [h for h in old if self.alive[h] and h != new_root and self.descends(h, new_root)]
            surv.sort(key=lambda h: (-self.score[h], self.token[h], h))
            surv = surv[: self.K]
        self.frontier = surv
        self._rebase()
        self.epoch += 1
        self._maybe_compact()
        return self.root

    def advance_root(self, accepted, corr) -> bool:    # cache.py:415-437
        chain = self.walk(accepted)
        anchor = chain[-1] if chain else self.root
        if corr is None:
            if not chain:
                raise OracleInputError("need a chain or a correction token")
            new_root = anchor
        else:
            new_root = self.child_with(anchor, int(corr))
            if new_root is None:
                return False
        self.root = new_root
        self.frontier = [h for h in self.frontier if self.alive[h]]
        self.epoch += 1
        return True

    def reset(self, root_token):                       # cache.py:439-444
        self._init_root(root_token)
        self.epoch += 1

    def _rebase(self):                                 # cache.py:454-469
        base = self.score[self.root]
        if base == 0.0:
            return
        stack = [self.root]
        while stack:
            h = stack.pop()
            self.score[h] = self.score[h] - base
            stack.extend(self.alive_children(h))
        self.score[self.root] = 0.0

    def _maybe_compact(self):                          # cache.py:471-504
        n = len(self.token)
        if n < COMPACT_MIN_ARENA or self.dead <= COMPACT_DEAD_FRACTION * n:
            return
        keep, stack = [], [self.root]
        while stack:
            h = stack.pop()
            keep.append(h)
            stack.extend(self.alive_children(h))
        keep.sort()
        remap = {old: new for new, old in enumerate(keep)}
        self.parent = [(-1 if (old == self.root or self.parent[old] not in remap)
                        else remap[self.parent[old]]) for old in keep]
        self.token = [self.token[o] for o in keep]
        self.layer = [self.layer[o] for o in keep]
        self.score = [self.score[o] for o in keep]
        self.edge = [self.edge[o] for o in keep]
        self.alive = [True] * len(keep)
        self.kids = [[] for _ in keep]
        for h, p in enumerate(self.parent):
            if p >= 0:
                self.kids[p].append(h)
        self.root = remap[self.root]
        self.frontier = [remap[h] for h in self.frontier]
        self.dead = 0

    def dump(self) -> str:                             # cache.py:510-523
        lines = []

        def emit(h, depth):
            lines.append("  " * depth + f"{self.token[h]}:{self.score[h]:.6f}")
            kids = sorted(self.alive_children(h), key=lambda c: (self.token[c], c))
            for c in kids:
                emit(c, depth + 1)

        emit(self.root, 0)
        return "\n".join(lines) + "\n"


# --------------------------------------------------------------------------
# verification (verify.py:38-132)
# --------------------------------------------------------------------------

def argmax_token(p) -> int:
    return int(np.argmax(p))


def sample_index(rng, p) -> int:                       # verify.py:43-51
    cdf = np.cumsum(p)
    total = cdf[-1]
    if not np.isfinite(total) or total <= 0.0:
        raise OracleInputError("all-zero distribution")
    u = rng.random() * total
    return min(int(np.searchsorted(cdf, u, side="right")), len(p) - 1)


def verify_greedy(dists, cand):                        # verify.py:65-80
    n = 0
    while n < len(cand) and argmax_token(dists[n]) == cand[n]:
        n += 1
    return tuple(int(t) for t in cand[:n]), argmax_token(dists[n])


def verify_sampling(dists, q, cand, rng):              # verify.py:83-132
    n, corr = 0, None
    for i, tok in enumerate(cand):
        p = dists[i]
        qi = float(q[i])
        if not np.isfinite(qi) or qi <= 0.0:
            raise OracleProtocolError("zero draft conditional")
        if rng.random() < min(1.0, float(p[tok]) / qi):
            n += 1
            continue
        oh = np.zeros(len(p))
        oh[tok] = 1.0
        resid = np.maximum(p - qi * oh, 0.0)
        if float(resid.sum()) <= 0.0:
            resid = p
        corr = sample_index(rng, resid)
        break
    if corr is None:
        corr = sample_index(rng, dists[len(cand)])
    return tuple(int(t) for t in cand[:n]), corr


# --------------------------------------------------------------------------
# models: the ToyModel protocol (lm.py:109-196) for the k-gram toy
# --------------------------------------------------------------------------

@dataclass
class OracleKGram:
    seed: int
    vocab_size: int
    order: int
    sharpness: float
    params_billions: float = 1.0
    forward_latency: float = 1.0
    eos_token: int | None = None
    mix_seed: int = 0
    mix_weight: float = 0.0
    _memo: dict = field(default_factory=dict, repr=False)

    def next_distribution(self, ctx, temperature=1.0):   # lm.py:140-153, 234-256
        ctx = tuple(int(t) for t in ctx)
        if self.eos_token is not None and ctx[-1] == self.eos_token:
            out = np.zeros(self.vocab_size)
            out[self.eos_token] = 1.0
            return out
        key = (ctx[-self.order:], float(temperature))
        hit = self._memo.get(key)
        if hit is None:
            hit = kgram_dist(self.seed, self.mix_seed, self.mix_weight, key[0],
                             self.vocab_size, self.sharpness, float(temperature))
            self._memo[key] = hit
        return hit


def load_pair(doc: dict):
    """Models JSON (lm.py:438-464, kgram/uniform only)."""
    V = doc["vocab_size"]
    eos = doc.get("eos_token")

    def build(c):
        kind = c.get("type", "kgram")
        if kind == "uniform":
            return OracleKGram(0, V, 1, 0.0, c.get("params_billions", 1.0),
                               c.get("forward_latency", 1.0), eos)
        return OracleKGram(c.get("seed", 0), V, c.get("order", 2), c.get("sharpness", 1.0),
                           c.get("params_billions", 1.0), c.get("forward_latency", 1.0), eos,
                           c.get("mix_seed", 0), c.get("mix_weight", 0.0))

    return build(doc["draft"]), build(doc["target"])


# --------------------------------------------------------------------------
# serial engine (engine.py:149-317, 392-423) and metrics (metrics.py:52-149)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Event:
    step_index: int
    sim_time: float
    hit: bool
    candidate_len: int
    accepted_len: int
    lnew: int
    cache_alive_nodes: int
    event: str


def run_serial(draft, target, prompt, K=50, k=3, ratio=5, temperature=0.0, max_new_tokens=64,
               correction_enabled=True, seed=0, query_depth=None, max_depth=None):
    """Deterministic lockstep schedule (engine.py:290-317).  Returns
    (output tokens, list[Event])."""
    res = None
    for res in serial_cycles(draft, target, prompt, K, k, ratio, temperature, max_new_tokens, correction_enabled,
                             seed, query_depth, max_depth):
        pass
    return res


def serial_cycles(draft, target, prompt, K=50, k=3, ratio=5, temperature=0.0, max_new_tokens=64,
                  correction_enabled=True, seed=0, query_depth=None, max_depth=None):
    """run_serial as a generator: yields (output, trace) after the warm-up
    expansions and after every cycle (the bench's bounded CPU samples)."""
    qd = ratio if query_depth is None else query_depth
    md = 2 * ratio if max_depth is None else max_depth
    prompt = [int(t) for t in prompt]
    t_score = temperature if temperature > 0.0 else 1.0
    sampling = temperature > 0.0
    rng = np.random.default_rng(seed)
    eos = target.eos_token
    tree = SoATree(prompt[-1], K, k, md, eos)
    anchor_origin = not correction_enabled           # engine.py:171-174
    out: list[int] = []
    trace: list[Event] = []
    st = {"base": list(prompt), "done": False}

    def committed():
        return prompt + out

    def emit(t, hit, cl, al, ln, ev):
        trace.append(Event(len(trace), t, hit, cl, al, ln, tree.alive_below_root(), ev))

    def draft_step():                                  # engine.py:198-221
        if tree.frontier:
            anc = 0 if anchor_origin else tree.root
            paths = [[tree.token[x] for x in tree.path_to(h, anc)] for h in tree.frontier]
            if hasattr(draft, "tree_distributions") and all(paths):   # one masked pass (lm.py:155-163)
                dists = draft.tree_distributions(st["base"], paths, t_score)
            else:
                dists = [draft.next_distribution(st["base"] + p, t_score) for p in paths]
        else:
            dists = [draft.next_distribution(committed(), t_score)]
        try:
            new = tree.expand(np.vstack(dists))
        except OracleFrontierFull:
            return 0
        return len(new)

    def target_step():                                 # engine.py:228-245
        hit, _, toks, _ = tree.query(qd)
        if not hit:
            d = target.next_distribution(committed(), t_score)
            tok = sample_index(rng, d) if sampling else argmax_token(d)
            return False, 0, (), tok
        ctx = committed()
        if hasattr(target, "chain_distributions"):   # the chain in one pass
            dists = target.chain_distributions(ctx, list(toks), t_score)
        else:
            dists = [target.next_distribution(ctx + toks[:i], t_score) for i in range(len(toks) + 1)]
        if sampling:
            acc, corr = verify_sampling(dists, [1.0] * len(toks), toks, rng)
        else:
            acc, corr = verify_greedy(dists, toks)
        return True, len(toks), acc, corr

    def commit(acc, corr):                             # engine.py:247-262
        lnew = len(acc) + 1
        room = max_new_tokens - len(out)
        toks = (list(acc) + [corr])[:room]
        if eos is not None and eos in toks:
            toks = toks[: toks.index(eos) + 1]
        out.extend(toks)
        if len(toks) < lnew or len(out) >= max_new_tokens:
            st["done"] = True
        if toks and eos is not None and toks[-1] == eos:
            st["done"] = True
        return max(0, len(toks) - 1), len(toks)

    def update(acc, corr):                             # engine.py:264-272
        if correction_enabled:
            tree.correct(list(acc), corr)
            st["base"] = committed()
        elif not tree.advance_root(list(acc), corr):
            tree.reset(out[-1])
            st["base"] = committed()

    d_lat, t_lat = draft.forward_latency, target.forward_latency
    clock = 0.0
    for _ in range(qd):
        w = draft_step()
        if w == 0:
            break
        clock += d_lat
        emit(clock, False, w, 0, 0, "draft_expand")
    yield out, trace
    while not st["done"]:
        start, n_exp = clock, 0
        for _ in range(ratio):
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
            update(acc, corr)
            emit(clock, hit, 0, 0, 0, "correct")
        yield out, trace


def run_vanilla(target, prompt, temperature=0.0, max_new_tokens=64, seed=0):
    """engine.py:392-423"""
    toks = [int(t) for t in prompt]
    t_score = temperature if temperature > 0.0 else 1.0
    rng = np.random.default_rng(seed)
    out, trace, clock = [], [], 0.0
    while len(out) < max_new_tokens:
        d = target.next_distribution(toks + out, t_score)
        tok = sample_index(rng, d) if temperature > 0.0 else argmax_token(d)
        out.append(tok)
        clock += target.forward_latency
        trace.append(Event(len(trace), clock, False, 0, 0, 1, 0, "miss_step"))
        if target.eos_token is not None and tok == target.eos_token:
            break
    return out, trace


METRIC_FIELDS = ("tokens_emitted", "sim_time", "target_forwards", "draft_forwards", "hits",
                 "misses", "mean_acceptance_length", "cache_hit_rate", "tokens_per_time",
                 "speedup_vs_vanilla", "params_x_lnew", "draft_params_x_width")


def finalize(trace, t_params, t_lat, d_params=None) -> dict:
    """metrics.py:52-109"""
    tokens = tf = df = hits = misses = width = 0
    sim = 0.0
    for ev in trace:
        sim = max(sim, ev.sim_time)
        if ev.event in ("verify", "miss_step"):
            tf += 1
            tokens += ev.lnew
            hits += ev.event == "verify"
            misses += ev.event == "miss_step"
        elif ev.event == "draft_expand":
            df += 1
            width += ev.candidate_len
    mean = tokens / tf
    q = hits + misses
    return dict(tokens_emitted=tokens, sim_time=sim, target_forwards=tf, draft_forwards=df,
                hits=hits, misses=misses, mean_acceptance_length=mean,
                cache_hit_rate=hits / q if q else 0.0,
                tokens_per_time=tokens / sim if sim > 0 else 0.0,
                speedup_vs_vanilla=(tokens * t_lat) / sim if sim > 0 else 0.0,
                params_x_lnew=t_params * mean,
                draft_params_x_width=(d_params or 0.0) * (width / df if df else 0.0))


def aggregate(runs) -> dict:
    """metrics.py:112-149"""
    runs = list(runs)
    s = lambda f: sum(r[f] for r in runs)  # noqa: E731
    tokens, sim, tf, df = s("tokens_emitted"), s("sim_time"), s("target_forwards"), s("draft_forwards")
    hits, misses = s("hits"), s("misses")
    vanilla = sum(r["speedup_vs_vanilla"] * r["sim_time"] for r in runs)
    pxl = sum(r["params_x_lnew"] * r["target_forwards"] for r in runs)
    dxw = sum(r["draft_params_x_width"] * r["draft_forwards"] for r in runs)
    q = hits + misses
    return dict(tokens_emitted=tokens, sim_time=sim, target_forwards=tf, draft_forwards=df,
                hits=hits, misses=misses,
                mean_acceptance_length=tokens / tf if tf else 0.0,
                cache_hit_rate=hits / q if q else 0.0,
                tokens_per_time=tokens / sim if sim > 0 else 0.0,
                speedup_vs_vanilla=vanilla / sim if sim > 0 else 0.0,
                params_x_lnew=pxl / tf if tf else 0.0,
                draft_params_x_width=dxw / df if df else 0.0)
