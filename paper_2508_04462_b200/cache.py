"""Device-resident candidate tree — drop-in for ``specache.cache``
(/root/reference/pkg/src/specache/cache.py:34-523).

The tree lives in HBM as a struct-of-arrays arena (see
csrc/card_cache.cu); every mutating operation and every query is one CUDA
kernel behind the C-ABI.  This class is the synchronous, reference-shaped
facade: it launches the kernel on the current stream, reads the status
word back and raises the reference's exception types.  Read-side helpers
(``arena``, ``dump``, ``path_from_root`` …) are views over a snapshot of
the device arrays.  The engine drives the same handle asynchronously.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from ._device import ptr, require_cuda, stream_ptr, to_device
from ._lib import CacheState, lib
from .errors import ConfigError, FrontierFull, InputError, raise_for_status

TokenId = int


@dataclass
class CacheConfig:
    """Beam geometry: K frontier slots, k extensions per node, depth cap (cache.py:34-46)."""

    K: int
    k: int
    max_depth: int

    def __post_init__(self):
        for name in ("K", "k", "max_depth"):
            v = getattr(self, name)
            if not isinstance(v, int) or isinstance(v, bool) or v < 1:
                raise ConfigError(f"CacheConfig.{name} must be an int >= 1, got {v!r}")


@dataclass
class CacheNode:
    node_id: int
    token: TokenId
    parent: int | None
    layer: int
    log_score: float
    edge_logp: float
    alive: bool = True
    children: list[int] = field(default_factory=list)


@dataclass(frozen=True)
class CandidateTuple:
    token: TokenId
    weight: float
    parent_index: int
    edge_logp: float = 0.0


@dataclass
class QueryResult:
    hit: bool
    path: list[int]
    tokens: list[TokenId]
    edge_logps: list[float]

    @property
    def conditionals(self) -> list[float]:
        return [math.exp(e) for e in self.edge_logps]


class TreeCache:
    """Drop-in TreeCache over the device arena (cache.py:92-523)."""

    def __init__(self, root_token: TokenId, config: CacheConfig, eos_token: TokenId | None = None,
                 capacity: int | None = None):
        if not isinstance(root_token, (int, np.integer)) or isinstance(root_token, bool) or root_token < 0:
            raise InputError(f"root token must be a non-negative int, got {root_token!r}")
        self.config = config
        self.eos_token = eos_token
        self._dev = require_cuda()
        h = ctypes.c_void_p()
        rc = lib().card_cache_create(int(root_token), config.K, config.k, config.max_depth,
                                     -1 if eos_token is None else int(eos_token),
                                     int(capacity or 0), ctypes.byref(h))
        raise_for_status(rc, "card_cache_create")
        self._h = h
        md = config.max_depth + 2
        self._acc = torch.zeros(md, dtype=torch.int32, device=self._dev)
        self._nacc = torch.zeros(1, dtype=torch.int32, device=self._dev)
        self._corr = torch.zeros(1, dtype=torch.int32, device=self._dev)
        qp, qt, qe = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        lib().card_cache_query_buffers(h, ctypes.byref(qp), ctypes.byref(qt), ctypes.byref(qe))
        self._qbufs = (qp.value, qt.value, qe.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                torch.cuda.synchronize()
                lib().card_cache_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    # ------------------------------------------------------------ state reads
    def state(self) -> CacheState:
        st = CacheState()
        raise_for_status(lib().card_cache_read_state(self._h, ctypes.byref(st), stream_ptr()), "read_state")
        return st

    @property
    def epoch(self) -> int:
        return self.state().epoch

    @property
    def root(self) -> int:
        return self.state().root

    @property
    def frontier(self) -> list[int]:
        return self._snapshot()["frontier"]

    def _snapshot(self) -> dict:
        st = self.state()
        n, f = st.n_nodes, st.n_frontier
        tok = np.empty(n, np.int32)
        par = np.empty(n, np.int32)
        lay = np.empty(n, np.int32)
        alv = np.empty(n, np.uint8)
        sc = np.empty(n, np.float64)
        ed = np.empty(n, np.float64)
        fr = np.empty(max(f, 1), np.int32)
        c = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        rc = lib().card_cache_snapshot(self._h, c(tok), c(par), c(lay), c(alv), c(sc), c(ed), c(fr), stream_ptr())
        raise_for_status(rc, "snapshot")
        return dict(state=st, token=tok.tolist(), parent=par.tolist(), layer=lay.tolist(),
                    alive=[bool(x) for x in alv], score=sc.tolist(), edge=ed.tolist(),
                    frontier=fr[:f].tolist(), root=st.root, epoch=st.epoch, dead=st.dead)

    @property
    def arena(self) -> list[CacheNode]:
        s = self._snapshot()
        nodes = [CacheNode(node_id=i, token=s["token"][i], parent=(None if s["parent"][i] < 0 else s["parent"][i]),
                           layer=s["layer"][i], log_score=s["score"][i], edge_logp=s["edge"][i],
                           alive=s["alive"][i]) for i in range(len(s["token"]))]
        for nd in nodes:
            if nd.parent is not None:
                nodes[nd.parent].children.append(nd.node_id)
        return nodes

    def node(self, handle: int) -> CacheNode:
        return self.arena[handle]

    def depth_below_root(self) -> int:
        s = self._snapshot()
        if not s["frontier"]:
            return 0
        return s["layer"][s["frontier"][0]] - s["layer"][s["root"]]

    def expansion_parents(self) -> list[int]:
        s = self._snapshot()
        return list(s["frontier"]) if s["frontier"] else [s["root"]]

    def path_from_root(self, handle: int) -> list[int]:
        s = self._snapshot()
        from .errors import ProtocolError

        rev, cur = [], handle
        while cur != s["root"]:
            rev.append(cur)
            cur = s["parent"][cur]
            if cur < 0:
                raise ProtocolError(f"node {handle} does not descend from the current root")
        return rev[::-1]

    def parent_paths(self) -> list[list[TokenId]]:
        s = self._snapshot()
        out = []
        for h in (s["frontier"] or [s["root"]]):
            rev, cur = [], h
            while cur != s["root"]:
                rev.append(s["token"][cur])
                cur = s["parent"][cur]
            out.append(rev[::-1])
        return out

    def alive_below_root(self) -> int:
        raise_for_status(lib().card_cache_count_alive(self._h, stream_ptr()), "count_alive")
        return self.state().alive_below

    # ------------------------------------------------------------ expansion
    def extension_pool(self, distributions) -> list[CandidateTuple]:
        """cache.py:190-222 — device row top-k + correctly rounded log."""
        d = np.asarray(distributions, dtype=np.float64)
        parents = self.expansion_parents()
        if d.ndim != 2 or d.shape[0] != len(parents):
            raise InputError(f"expected {len(parents)} distributions, got array of shape {d.shape}")
        dev = to_device(d, np.float64)
        P = d.shape[0] * self.config.k
        tok = torch.empty(P, dtype=torch.int32, device=self._dev)
        w = torch.empty(P, dtype=torch.float64, device=self._dev)
        pidx = torch.empty(P, dtype=torch.int32, device=self._dev)
        e = torch.empty(P, dtype=torch.float64, device=self._dev)
        lib().card_cache_clear_status(self._h, stream_ptr())
        rc = lib().card_cache_pool(self._h, ptr(dev), d.shape[0], d.shape[1], ptr(tok), ptr(w), ptr(pidx), ptr(e),
                                   stream_ptr())
        raise_for_status(rc, "card_cache_pool")
        raise_for_status(self.state().vstatus, "extension_pool")
        tok, w, pidx, e = (x.cpu().tolist() for x in (tok, w, pidx, e))
        return [CandidateTuple(token=t, weight=ww, parent_index=pi, edge_logp=ee)
                for t, ww, pi, ee in zip(tok, w, pidx, e) if t >= 0]

    def expand_layer(self, distributions) -> list[int]:
        """cache.py:224-251 on the device."""
        d = np.asarray(distributions, dtype=np.float64)
        if d.ndim != 2:
            if self.depth_below_root() >= self.config.max_depth:
                raise FrontierFull(f"candidate tree already {self.config.max_depth} layers deep")
            raise InputError(f"expected a 2-D array of distributions, got shape {d.shape}")
        dev = to_device(d, np.float64)
        lib().card_cache_clear_status(self._h, stream_ptr())
        rc = lib().card_cache_expand(self._h, ptr(dev), d.shape[0], d.shape[1], stream_ptr())
        raise_for_status(rc, "card_cache_expand")
        st = self.state()
        if st.status == -4:
            raise FrontierFull(f"candidate tree already {self.config.max_depth} layers deep")
        raise_for_status(st.status, "expand_layer")
        return self.frontier

    # ------------------------------------------------------------ query
    def query(self, depth: int) -> QueryResult:
        """cache.py:277-318 on the device."""
        if not isinstance(depth, int) or isinstance(depth, bool) or depth < 1:
            raise InputError(f"query depth must be an int >= 1, got {depth!r}")
        raise_for_status(lib().card_cache_query(self._h, depth, stream_ptr()), "card_cache_query")
        st = self.state()
        raise_for_status(st.status, "query")
        if not st.q_hit:
            return QueryResult(hit=False, path=[], tokens=[], edge_logps=[])
        n = st.q_len
        qp, qt, qe = self._qbufs
        path = device_view(qp, np.int32, n).tolist() if n else []
        toks = device_view(qt, np.int32, n).tolist() if n else []
        edges = device_view(qe, np.float64, n).tolist() if n else []
        return QueryResult(hit=True, path=path, tokens=toks, edge_logps=edges)

    # ------------------------------------------------------------ correction
    def _load_commit(self, accepted, correction_token):
        acc = [int(t) for t in accepted]
        if len(acc) > self._acc.numel():
            acc = acc[: self._acc.numel()]   # longer than any cached chain: the walk fails on device
            over = True
        else:
            over = False
        if acc:
            self._acc[: len(acc)].copy_(torch.tensor(acc, dtype=torch.int32))
        self._nacc.fill_(len(acc) if not over else self._acc.numel())
        self._corr.fill_(-1 if correction_token is None else int(correction_token))

    def correct(self, accepted, correction_token: TokenId | None) -> int:
        """cache.py:355-413 on the device."""
        self._load_commit(accepted, correction_token)
        rc = lib().card_cache_correct(self._h, ptr(self._acc), ptr(self._nacc), ptr(self._corr), None, stream_ptr())
        raise_for_status(rc, "card_cache_correct")
        st = self.state()
        raise_for_status(st.status, "correct")
        return st.root

    def advance_root(self, accepted, correction_token: TokenId | None) -> bool:
        """cache.py:415-437 on the device."""
        self._load_commit(accepted, correction_token)
        rc = lib().card_cache_advance_root(self._h, ptr(self._acc), ptr(self._nacc), ptr(self._corr), stream_ptr())
        raise_for_status(rc, "card_cache_advance_root")
        st = self.state()
        raise_for_status(st.status, "advance_root")
        return bool(st.moved)

    def clear(self, root_token: TokenId) -> None:
        """Back to the freshly created state (new request on a reused arena)."""
        raise_for_status(lib().card_cache_clear(self._h, int(root_token), stream_ptr()), "clear")

    def reset(self, root_token: TokenId) -> None:
        """cache.py:439-444 on the device."""
        if not isinstance(root_token, (int, np.integer)) or root_token < 0:
            raise InputError(f"root token must be a non-negative int, got {root_token!r}")
        raise_for_status(lib().card_cache_reset(self._h, None, int(root_token), stream_ptr()), "reset")
        raise_for_status(self.state().status, "reset")

    # ------------------------------------------------------------ debug
    def dump(self) -> str:
        """Deterministic pre-order rendering of the alive tree (cache.py:510-523)."""
        s = self._snapshot()
        kids: dict[int, list[int]] = {}
        for i, p in enumerate(s["parent"]):
            if p >= 0 and s["alive"][i]:
                kids.setdefault(p, []).append(i)
        lines: list[str] = []

        def emit(h, depth):
            lines.append("  " * depth + f"{s['token'][h]}:{s['score'][h]:.6f}")
            for c in sorted(kids.get(h, []), key=lambda c: (s["token"][c], c)):
                emit(c, depth + 1)

        emit(s["root"], 0)
        return "\n".join(lines) + "\n"


def device_view(addr: int, dtype, n: int) -> torch.Tensor:
    """Borrowed torch view of n elements of library-owned device memory."""
    dt = np.dtype(dtype)

    class _Iface:
        __cuda_array_interface__ = {"shape": (n,), "typestr": dt.str, "data": (addr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_Iface(), device="cuda")
