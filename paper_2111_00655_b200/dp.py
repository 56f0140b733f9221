"""Operator-level placement search (API of tensorplace/dp.py), solved on the
GPU by cb_dp_solve (csrc/dp.cu).

The reference DP (Algorithm 1) relaxes every stored covered-set state for
every candidate match in frontier order; its optimum is the cheapest
partition of the graph into registered matches under the additive model,
with ties broken by the canonical key (registration index, sorted node ids).
Because a match only exposes its root, the kernels of every partition nest
along the post-dominator tree, so the device solves the same problem as an
exact DP over post-dominator subtrees, one warp per node and one
topological level at a time (see csrc/dp.cu).  Results -- cost, kernels
and tie-breaking -- are those of the reference; only the search-internal
counters differ (the device examines each candidate exactly once, so
`relaxations` equals the number of candidates and the live state count is
the node count + 1).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from typing import Any, Mapping

import numpy as np

from . import _native as nat
from .cost import Measurer, price_matches
from .errors import RoundingWindowError, SearchLimitError, UncoverableGraphError
from .graph import ComputationGraph
from .placement import Assignment, PlacementStrategy, validate_placement
from .registry import PatternRegistry

DEFAULT_MAX_STATES = None  # the subtree DP has n + 1 states; no cap needed
VALIDATE_MAX_NODES = 5000


@dataclass
class DPStats:
    nodes: int = 0
    pops: int = 0
    candidates_total: int = 0
    max_candidates: int = 0
    max_new_frontiers: int = 0
    max_compatible_states: int = 0
    relaxations: int = 0
    improvements: int = 0
    measure_calls: int = 0
    cache_hits: int = 0
    computations: int = 0
    states_peak: int = 0

    # measure_calls / cache_hits / computations of a device pricing pass are
    # settled when first read (the reference's per-candidate cache protocol
    # is replayed lazily, see cost._account)
    def __getattribute__(self, name: str):
        if name in _LAZY_COUNTERS:
            d = object.__getattribute__(self, "__dict__")
            settle = d.pop("_settle", None)
            if settle is not None:
                settle(self)
        return object.__getattribute__(self, name)

    def to_json(self) -> dict:
        self.measure_calls  # settle
        return {k: v for k, v in self.__dict__.items() if not k.startswith("_")}

    def __getstate__(self) -> dict:  # pickling settles the lazy counters first
        return self.to_json()


_LAZY_COUNTERS = frozenset(("measure_calls", "cache_hits", "computations"))


@dataclass
class DPResult:
    placement: PlacementStrategy
    cost_ms: float
    stats: DPStats
    state_costs: Mapping[frozenset, float] = field(default_factory=dict)
    device: dict[str, Any] = field(default_factory=dict)
    kernel_matches: np.ndarray | None = None  # match-table indices, canonical order


def _new_frontiers(g: ComputationGraph) -> int:
    """Largest number of nodes first enqueued by a single pop (pop order is
    (depth, id)); mirrors the reference counter (vectorised over the CSR)."""
    n = len(g.nodes)
    if n == 0:
        return 0
    order = np.lexsort((np.arange(n), g._depth_arr))  # pop order over node indices
    rank = np.empty(n, dtype=np.int64)
    rank[order] = np.arange(n)
    src = g._in_src.astype(np.int64)
    dst = np.repeat(np.arange(n), np.diff(g._in_ptr))
    keep = src >= 0
    src, dst = src[keep], dst[keep]
    if src.size == 0:
        return 0
    # for every consumer, the predecessor that pops first enqueues it
    best = np.full(n, np.iinfo(np.int64).max)
    np.minimum.at(best, dst, rank[src])
    firsts = best[best != np.iinfo(np.int64).max]
    return int(np.bincount(firsts).max())


def optimize(g: ComputationGraph, registry: PatternRegistry, measurer: Measurer,
             epsilon: float, max_states: int | None = DEFAULT_MAX_STATES,
             validate: bool | None = None, rounding: str = "raise",
             stream: int | None = None) -> DPResult:
    """Cheapest full placement of `g` (exact, reference tie-breaking).

    Raises UncoverableGraphError when no full cover exists and
    SearchLimitError when `max_states` is given and the n + 1 subtree states
    exceed it.  The device compares exact sums; the reference compares
    rounded ones.  When the solver cannot certify that both choose the same
    partition (an alternative within 4 ulp of the total, see csrc/dp.cu
    rounding_window_safe), `rounding="raise"` (default) raises
    RoundingWindowError carrying the exact result, `rounding="exact"`
    returns the exact optimum (`device["rounding_window_safe"]` False).
    `stream` (a cudaStream_t as int, e.g. torch's `cuda_stream`) runs the DP
    launches there instead of the legacy default stream."""
    if rounding not in ("raise", "exact"):
        raise ValueError("rounding must be 'raise' or 'exact'")
    stats = DPStats(nodes=len(g.nodes))
    c0, h0, p0 = measurer.calls, measurer.cache_hits, measurer.computations
    if not g.nodes:
        return DPResult(PlacementStrategy(()), 0.0, stats, {frozenset(): 0.0})
    uncovered = registry.uncovered_op_kinds(g)
    if uncovered:
        raise UncoverableGraphError(
            f"no registered pattern can root op kind(s) {list(uncovered)}", op_kinds=uncovered)
    if max_states is not None and len(g.nodes) + 1 > max_states:
        raise SearchLimitError(f"operator-level search needs {len(g.nodes) + 1} live states on "
                               f"a {len(g.nodes)}-node graph, above the cap of {max_states}")
    t0 = time.perf_counter()
    table = registry.match_table(g)
    t1 = time.perf_counter()
    price_matches(measurer, registry, table)
    t2 = time.perf_counter()
    kernels = np.empty(len(g.nodes), dtype=np.int32)
    res = nat.DPResultStruct()
    nat.check(nat.lib().cb_dp_solve_stream(g.native, table.handle.raw, float(epsilon),
                                           nat.ptr(kernels, nat.c_int32), ctypes.byref(res),
                                           ctypes.c_void_p(stream or 0)))
    t3 = time.perf_counter()
    sizes = np.diff(table.group_ptr)
    stats.pops = len(g.nodes)
    stats.candidates_total = int(table.n_matches)
    stats.max_candidates = int(sizes.max()) if len(sizes) else 0
    stats.max_new_frontiers = _new_frontiers(g)
    stats.max_compatible_states = 1 if table.n_matches else 0
    stats.relaxations = int(table.n_matches)
    stats.states_peak = len(g.nodes) + 1
    acct = getattr(table, "_account", None)
    if acct is not None and getattr(table, "_priced", (None,))[0] is measurer:
        # device pricing: this pass's share of the reference's cache protocol,
        # settled (replayed) when a counter is first read
        def settle(st, acct=acct, cache=measurer.cache):
            cache._flush()
            st.measure_calls = acct.get("calls", 0)
            st.cache_hits = acct.get("cache_hits", 0)
            st.computations = acct.get("computations", 0)
        stats.__dict__["_settle"] = settle
    else:
        stats.measure_calls = measurer.calls - c0
        stats.cache_hits = measurer.cache_hits - h0
        stats.computations = measurer.computations - p0
    device = {"device_ms": res.device_ms, "levels": res.n_levels, "launches": res.n_launches,
              "ties": res.ties, "walk_steps": res.walk_steps,
              "rounding_window_safe": bool(res.window_safe),
              "phases_s": {"match": t1 - t0, "price": t2 - t1, "dp_call": t3 - t2}}
    if not res.feasible:
        z = res.first_zero_candidate
        if z >= 0:
            nid = g.id_of(z)
            kind = g.nodes[nid].op_kind
            raise UncoverableGraphError(
                f"no full placement found; frontier node {nid} (op '{kind}') had zero "
                f"candidate matches", op_kinds=(kind,), node_ids=(nid,))
        raise UncoverableGraphError("no full placement found; some nodes cannot be covered "
                                    "compatibly by the registered patterns")
    chosen = kernels[:res.n_kernels]
    # canonical order (sorted node tuple): the kernels are disjoint, so it is
    # the order of their smallest members (member lists are sorted, node
    # indices follow node ids) -- vectorised; the Assignment objects are
    # built only when the placement's assignments are first read
    first = table.members[table.mem_ptr[chosen]] if len(chosen) else np.zeros(0, np.int64)
    canon = np.ascontiguousarray(chosen[np.argsort(first, kind="stable")], dtype=np.int32)
    patterns = registry.patterns

    def build() -> list[Assignment]:
        ms = canon.tolist()
        sets = table.node_sets(ms)
        pats = table.pat[canon].tolist()
        roots = np.asarray(g._ids)[table.root[canon]].tolist()
        return [Assignment.fast(sets[i], patterns[pats[i]], roots[i]) for i in range(len(ms))]

    stats.improvements = len(g.nodes)  # every node's subtree optimum is set once
    placement = PlacementStrategy.lazy(len(canon), build)
    t4 = time.perf_counter()
    if validate or (validate is None and len(g.nodes) <= VALIDATE_MAX_NODES):
        validate_placement(g, placement)
    device["phases_s"].update(result=t4 - t3, validate=time.perf_counter() - t4)
    out = DPResult(placement, res.cost_ms, stats,
                   {frozenset(g.nodes): res.cost_ms, frozenset(): 0.0}, device, canon)
    if not device["rounding_window_safe"] and rounding == "raise":
        raise RoundingWindowError(
            f"an alternative placement differs from the exact optimum ({res.cost_ms!r} ms) by "
            f"less than the rounding resolution of the total; the reference's rounded "
            f"comparisons may pick either (pass rounding='exact' to accept the exact optimum)",
            out)
    return out
