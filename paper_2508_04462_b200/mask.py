"""Tree-attention visibility (drop-in for ``specache.mask``,
/root/reference/pkg/src/specache/mask.py:31-217).

The device never materialises this mask: the draft row builder
(``csrc/card_engine.cu`` ``draft_rows_kernel``) gives every frontier row its
ancestor chain as a list of KV slots, and the tree attention reads exactly
those.  This module is the boolean form of the same relation for callers of
the reference API (``ToyModel.batch_tree_forward`` consumers, differential
tests).  It works on a snapshot of any tree that exposes the arena as
parent/token/layer/alive arrays: the device ``TreeCache`` (one
``card_cache_snapshot`` per call), the oracle ``SoATree``, or a reference-
style ``arena`` of nodes.

Visibility of a node below an anchor (the cache root, or an explicit handle
for the un-steered ablation, mask.py:8-12) is its chain of ancestors
strictly below the anchor plus itself.  Arena ids grow monotonically and
compaction preserves order, so every parent id is smaller than its
children's: the "alive below the anchor" set is one pass in id order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InputError

TokenId = int


@dataclass
class AttentionMask:
    """Rows = the newest tree layer; columns = visible tree tokens, the last
    ``n_new`` of them being the new tokens (mask.py:31-49)."""

    bits: np.ndarray
    n_new: int
    columns: list[int]
    tokens: list[TokenId]

    def to_text(self) -> str:
        return "".join("".join("1" if b else "0" for b in row) + "\n" for row in np.asarray(self.bits))


class _Tree:
    """Immutable arrays of one tree snapshot."""

    __slots__ = ("parent", "token", "layer", "alive", "frontier", "root", "epoch")

    def __init__(self, parent, token, layer, alive, frontier, root, epoch):
        self.parent = np.asarray(parent, dtype=np.int64)
        self.token = [int(t) for t in token]
        self.layer = np.asarray(layer, dtype=np.int64)
        self.alive = np.asarray(alive, dtype=bool)
        self.frontier = [int(h) for h in frontier]
        self.root = int(root)
        self.epoch = int(epoch)

    @property
    def n(self) -> int:
        return len(self.token)

    def anchor(self, anchor: int | None) -> int:
        if anchor is None:
            return self.root
        if not isinstance(anchor, (int, np.integer)) or isinstance(anchor, bool) or not 0 <= anchor < self.n:
            raise InputError(f"unknown anchor handle {anchor!r}")
        if not self.alive[anchor]:
            raise InputError(f"anchor handle {anchor} is dead")
        return int(anchor)

    def below(self, anchor: int) -> list[int]:
        """Alive nodes reachable from the anchor through alive nodes, in
        (layer, id) order (mask.py:60-71)."""
        reach = np.zeros(self.n, dtype=bool)
        for h in range(anchor + 1, self.n):
            p = self.parent[h]
            if self.alive[h] and p >= 0 and (p == anchor or reach[p]):
                reach[h] = True
        hs = np.flatnonzero(reach)
        return [int(h) for h in hs[np.lexsort((hs, self.layer[hs]))]]

    def chain(self, h: int, anchor: int) -> list[int]:
        """Handles strictly below the anchor down to h, shallowest first."""
        out = []
        cur = int(h)
        while cur != anchor:
            if cur < 0:
                raise InputError(f"node {h} does not descend from anchor {anchor}")
            out.append(cur)
            cur = int(self.parent[cur])
        out.reverse()
        return out


def _tree(cache) -> _Tree:
    if hasattr(cache, "_snapshot"):          # device TreeCache
        s = cache._snapshot()
        return _Tree(s["parent"], s["token"], s["layer"], s["alive"], s["frontier"], s["root"], s["epoch"])
    if hasattr(cache, "parent") and hasattr(cache, "layer"):   # oracle SoATree
        return _Tree(cache.parent, cache.token, cache.layer, cache.alive, cache.frontier, cache.root,
                     getattr(cache, "epoch", 0))
    arena = cache.arena                       # reference-style node list
    return _Tree([-1 if n.parent is None else n.parent for n in arena], [n.token for n in arena],
                 [n.layer for n in arena], [n.alive for n in arena], cache.frontier, cache.root,
                 getattr(cache, "epoch", 0))


def build_mask(cache, new_tokens: list[tuple[int, TokenId]], anchor: int | None = None) -> AttentionMask:
    """Mask for hypothetical tokens attached at the given parents
    (mask.py:90-128): columns = every alive node below the anchor, then the
    new tokens; row i sees its parent's chain and its own column."""
    if not new_tokens:
        raise InputError("build_mask needs at least one (parent, token) pair")
    tr = _tree(cache)
    a = tr.anchor(anchor)
    prior = tr.below(a)
    col = {h: c for c, h in enumerate(prior)}
    n_new = len(new_tokens)
    bits = np.zeros((n_new, len(prior) + n_new), dtype=bool)
    for i, (parent, _tok) in enumerate(new_tokens):
        if not isinstance(parent, (int, np.integer)) or isinstance(parent, bool) or not 0 <= parent < tr.n:
            raise InputError(f"unknown parent handle {parent!r}")
        if not tr.alive[parent]:
            raise InputError(f"parent handle {parent} is dead")
        if parent != a:
            bits[i, [col[h] for h in tr.chain(parent, a)]] = True
        bits[i, len(prior) + i] = True
    return AttentionMask(bits=bits, n_new=n_new, columns=prior + [-1] * n_new,
                         tokens=[tr.token[h] for h in prior] + [int(t) for _, t in new_tokens])


def full_visibility(cache, anchor: int | None = None) -> tuple[list[int], np.ndarray]:
    """(handles in (layer, id) order, square ancestors-plus-self matrix) of
    the whole alive tree below the anchor (mask.py:131-148)."""
    tr = _tree(cache)
    a = tr.anchor(anchor)
    hs = tr.below(a)
    col = {h: c for c, h in enumerate(hs)}
    bits = np.zeros((len(hs), len(hs)), dtype=bool)
    for i, h in enumerate(hs):
        bits[i, [col[x] for x in tr.chain(h, a)]] = True
    return hs, bits


class MaskBuilder:
    """Frontier masks maintained across expansions (mask.py:151-217).

    A new node's visible chain is its parent's chain plus itself, so
    ``note_layer`` costs one lookup per new node.  Handles are only stable
    within one cache epoch: any correction, reset or compaction bumps the
    epoch and the next call rebuilds the chains from the tree."""

    def __init__(self, cache, anchor: int | None = None):
        self.cache = cache
        self._anchor_spec = anchor
        self._chains: dict[int, tuple[int, ...]] = {}
        self._epoch = None
        self._tree = None
        self._refresh()

    def _refresh(self) -> _Tree:
        tr = _tree(self.cache)
        if tr.epoch != self._epoch:
            a = tr.anchor(self._anchor_spec)
            self._chains = {h: tuple(tr.chain(h, a)) for h in tr.below(a)}
            self._epoch = tr.epoch
        self._tree = tr
        return tr

    def note_layer(self, new_handles: list[int]) -> None:
        """Record the chains of nodes an expansion just created."""
        tr = self._refresh()
        a = tr.anchor(self._anchor_spec)
        for h in new_handles:
            h = int(h)
            p = int(tr.parent[h])
            if p == a or p < 0:
                self._chains[h] = (h,)
                continue
            base = self._chains.get(p)
            if base is None:
                base = self._chains[p] = tuple(tr.chain(p, a))
            self._chains[h] = base + (h,)

    def frontier_mask(self) -> AttentionMask:
        """Columns: alive non-frontier nodes in (layer, id) order, then the
        frontier in frontier order (the trailing identity block)."""
        tr = self._refresh()
        a = tr.anchor(self._anchor_spec)
        front = tr.frontier
        if not front:
            raise InputError("cannot build a frontier mask for an empty frontier")
        fset = set(front)
        order = [h for h in tr.below(a) if h not in fset] + front
        col = {h: c for c, h in enumerate(order)}
        bits = np.zeros((len(front), len(order)), dtype=bool)
        for i, h in enumerate(front):
            ch = self._chains.get(h)
            if ch is None:
                ch = self._chains[h] = tuple(tr.chain(h, a))
            bits[i, [col[x] for x in ch]] = True
        return AttentionMask(bits=bits, n_new=len(front), columns=order, tokens=[tr.token[h] for h in order])
