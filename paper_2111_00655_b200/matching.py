"""Structural pattern matching (API of tensorplace/matching.py), executed by
the device matcher in libcollage_b200 (csrc/match.cu).

`match_at`, `match_all` and the registry's `candidates_at` all go through
the GPU: patterns are compiled to flat position tables, the device decides
every (anchor, pattern) pair with one warp per anchor and returns a
compacted CSR of matches that this module wraps in `Match` objects.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import PatternError
from .graph import ComputationGraph, Subgraph
from .patterns import CompiledPatterns, OpPattern, Pattern, Wildcard

Position = tuple[int, ...]


@dataclass(frozen=True)
class Match:
    """Pattern anchored at `root`: the op-bound nodes and the binding of
    every op position (argument-index path) to its node."""

    root: int
    nodes: Subgraph
    binding: tuple[tuple[Position, int], ...]

    def binding_map(self) -> dict[Position, int]:
        return dict(self.binding)


class NativePatterns:
    """A compiled pattern list uploaded to libcollage_b200."""

    def __init__(self, patterns: list[OpPattern], backends: list[int]):
        self.compiled = c = CompiledPatterns(patterns, backends)
        from ._encode import OP_KINDS
        n_kinds = len(OP_KINDS)
        order = np.argsort(c.root_kind, kind="stable") if c.n_pat else np.zeros(0, np.int64)
        kind_pat = nat.i32(order)
        counts = np.bincount(c.root_kind, minlength=n_kinds) if c.n_pat else np.zeros(n_kinds)
        kind_pat_ptr = nat.i32(np.concatenate([[0], np.cumsum(counts)]))
        raw = ctypes.c_void_p()
        L = nat.lib()
        I32, I8, I64, F64 = nat.c_int32, nat.c_int8, nat.c_int64, nat.c_double
        nat.check(L.cb_patterns_create(
            c.n_pat, n_kinds, nat.ptr(c.pos_ptr, I32), nat.ptr(c.kind, I32),
            nat.ptr(c.nargs, I32), nat.ptr(c.parent, I32), nat.ptr(c.argidx, I32),
            nat.ptr(c.sid, I32), nat.ptr(c.con_ptr, I32), nat.ptr(c.con_key, I32),
            nat.ptr(c.con_op, I8), nat.ptr(c.con_val_ptr, I32), nat.ptr(c.val_tag, I8),
            nat.ptr(c.val_ival, I64), nat.ptr(c.val_fval, F64), nat.ptr(c.con_lo, I64),
            nat.ptr(c.con_hi, I64), nat.ptr(c.backend, I32), nat.ptr(kind_pat_ptr, I32),
            nat.ptr(kind_pat, I32), ctypes.byref(raw)))
        self.handle = nat.Handle(raw.value, "cb_patterns_destroy")
        self._keep = (kind_pat, kind_pat_ptr)


class MatchTable:
    """Host view of a cb_matches object: matches grouped by `group` (the
    root node index for match_all, the pair index for match_pairs)."""

    def __init__(self, g: ComputationGraph, pats: NativePatterns, raw: int):
        self.graph = g
        self.patterns = pats
        self.handle = nat.Handle(raw, "cb_matches_destroy")
        L = nat.lib()
        ng, nm, nmem, nb = (ctypes.c_int64() for _ in range(4))
        nat.check(L.cb_matches_counts(self.handle.raw, ctypes.byref(ng), ctypes.byref(nm),
                                      ctypes.byref(nmem), ctypes.byref(nb)))
        self.n_groups, self.n_matches = ng.value, nm.value
        self.group_ptr = np.empty(ng.value + 1, np.int32)
        self.pat = np.empty(nm.value, np.int32)
        self.root = np.empty(nm.value, np.int32)
        self.mem_ptr = np.empty(nm.value + 1, np.int32)
        self.members = np.empty(nmem.value, np.int32)
        self.bind_ptr = np.empty(nm.value + 1, np.int32)
        self.binds = np.empty(nb.value, np.int32)
        I32 = nat.c_int32
        nat.check(L.cb_matches_download(
            self.handle.raw, nat.ptr(self.group_ptr, I32), nat.ptr(self.pat, I32),
            nat.ptr(self.root, I32), nat.ptr(self.mem_ptr, I32), nat.ptr(self.members, I32),
            nat.ptr(self.bind_ptr, I32), nat.ptr(self.binds, I32)))
        self._objs: dict[int, Match] = {}
        self._sets: dict[int, frozenset[int]] = {}
        self._lists = None

    @classmethod
    def all_anchors(cls, g: ComputationGraph, pats: NativePatterns) -> "MatchTable":
        nat.require_device()
        raw = ctypes.c_void_p()
        nat.check(nat.lib().cb_match_all(g.native, pats.handle.raw, ctypes.byref(raw)))
        return cls(g, pats, raw.value)

    @classmethod
    def pairs(cls, g: ComputationGraph, pats: NativePatterns, roots, pat_ids) -> "MatchTable":
        nat.require_device()
        r = nat.i32(roots)
        p = nat.i32(pat_ids)
        raw = ctypes.c_void_p()
        nat.check(nat.lib().cb_match_pairs(g.native, pats.handle.raw, len(r),
                                           nat.ptr(r, nat.c_int32), nat.ptr(p, nat.c_int32),
                                           ctypes.byref(raw)))
        return cls(g, pats, raw.value)

    def group(self, gi: int) -> range:
        return range(int(self.group_ptr[gi]), int(self.group_ptr[gi + 1]))

    def node_sets(self, ms: list[int]) -> list[frozenset[int]]:
        """node_set for many matches at once (no per-match cache lookups)."""
        if self._lists is None:
            self._lists = (self.members.tolist(), self.mem_ptr.tolist(),
                           np.asarray(self.graph._ids).tolist())
        mem, ptr, ids = self._lists
        return [frozenset([ids[v] for v in mem[ptr[m]:ptr[m + 1]]]) for m in ms]

    def node_set(self, m: int) -> frozenset[int]:
        s = self._sets.get(m)
        if s is None:
            if self._lists is None:  # Python-int views, built once per table
                self._lists = (self.members.tolist(), self.mem_ptr.tolist(),
                               np.asarray(self.graph._ids).tolist())
            mem, ptr, ids = self._lists
            s = frozenset([ids[v] for v in mem[ptr[m]:ptr[m + 1]]])
            self._sets[m] = s
        return s

    def match(self, m: int) -> Match:
        obj = self._objs.get(m)
        if obj is None:
            ids = self.graph._ids
            paths = self.patterns.compiled.paths[int(self.pat[m])]
            nodes = self.binds[self.bind_ptr[m]:self.bind_ptr[m + 1]]
            binding = tuple(sorted((paths[i], int(ids[v])) for i, v in enumerate(nodes)))
            obj = Match(root=int(ids[self.root[m]]),
                        nodes=Subgraph(self.graph, self.node_set(m)), binding=binding)
            self._objs[m] = obj
        return obj


_single_cache: dict[OpPattern, NativePatterns] = {}


def _single(pattern: OpPattern) -> NativePatterns:
    pats = _single_cache.get(pattern)
    if pats is None:
        pats = NativePatterns([pattern], [0])
        _single_cache[pattern] = pats
    return pats


def match_at(g: ComputationGraph, root_id: int, pattern: Pattern) -> Match | None:
    """Anchor `pattern` at node `root_id` (device matcher)."""
    if isinstance(pattern, Wildcard):
        raise PatternError("a bare wildcard cannot be matched as a full pattern")
    if root_id not in g.nodes:
        raise KeyError(f"unknown node id {root_id}")
    table = MatchTable.pairs(g, _single(pattern), [g.index_of(root_id)], [0])
    return table.match(0) if table.n_matches else None


def match_pairs(g: ComputationGraph, pairs: list[tuple[int, OpPattern]]) -> list[Match | None]:
    """Batched match_at over (root id, pattern) pairs in one device launch."""
    if not pairs:
        return []
    uniq: dict[OpPattern, int] = {}
    for _, p in pairs:
        if isinstance(p, Wildcard):
            raise PatternError("a bare wildcard cannot be matched as a full pattern")
        uniq.setdefault(p, len(uniq))
    pats = NativePatterns(list(uniq), [0] * len(uniq))
    roots = []
    for r, _ in pairs:
        if r not in g.nodes:
            raise KeyError(f"unknown node id {r}")
        roots.append(g.index_of(r))
    table = MatchTable.pairs(g, pats, roots, [uniq[p] for _, p in pairs])
    out: list[Match | None] = [None] * len(pairs)
    for i in range(len(pairs)):
        rng = table.group(i)
        if len(rng):
            out[i] = table.match(rng.start)
    return out


def match_all(g: ComputationGraph, pattern: Pattern) -> list[Match]:
    """Every match of `pattern`, by ascending root id (device matcher)."""
    if isinstance(pattern, Wildcard):
        raise PatternError("a bare wildcard cannot be matched as a full pattern")
    if not g.nodes:
        return []
    table = MatchTable.all_anchors(g, _single(pattern))
    return [table.match(m) for m in range(table.n_matches)]
