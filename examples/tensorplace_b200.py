"""Reference-side binding stub: what a `tensorplace` maintainer would add as
`tensorplace/_b200.py` to run the operator-level search on a B200 through
the C ABI of libcollage_b200.so (include/collage_b200.h).

It takes the reference's own objects -- a `ComputationGraph`, a
`PatternRegistry` and any `Measurer` -- and returns the placement of
`tensorplace.dp.optimize` (dp.py:71-179) as plain tuples.  Only the two
encoders come from this repo (graph CSR and pattern position tables); every
search call is a raw ctypes call into the library:

    cb_graph (via graph_from_json) -> cb_patterns_create -> cb_match_all
    -> cb_matches_download -> measurer.measure_kernel per match
    -> cb_matches_set_costs -> cb_dp_solve

`tests/test_integration_stub.py` runs it on the GPU and checks it against
`optimize`.
"""

from __future__ import annotations

import ctypes
import json
import os
from ctypes import POINTER, byref, c_double, c_int, c_int8, c_int32, c_int64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.environ.get("CB_LIB", os.path.join(HERE, "..", "paper_2111_00655_b200", "_lib",
                                               "libcollage_b200.so"))


class DPResult(ctypes.Structure):  # cb_dp_result
    _fields_ = [("cost_ms", c_double), ("feasible", c_int32), ("n_kernels", c_int32),
                ("n_levels", c_int32), ("n_launches", c_int32), ("candidates", c_int64),
                ("ties", c_int64), ("walk_steps", c_int64), ("window_safe", c_int32),
                ("first_zero_candidate", c_int32), ("device_ms", c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(LIB)
        P32, P8, P64, PF = POINTER(c_int32), POINTER(c_int8), POINTER(c_int64), POINTER(c_double)
        L.cb_last_error.restype = ctypes.c_char_p
        L.cb_patterns_create.argtypes = [c_int32, c_int32] + [P32] * 8 + [P8, P32, P8, P64, PF, P64,
                                                                          P64, P32, P32, P32,
                                                                          POINTER(c_void_p)]
        L.cb_match_all.argtypes = [c_void_p, c_void_p, POINTER(c_void_p)]
        L.cb_matches_counts.argtypes = [c_void_p] + [POINTER(c_int64)] * 4
        L.cb_matches_download.argtypes = [c_void_p] + [P32] * 7
        L.cb_matches_set_costs.argtypes = [c_void_p, PF]
        L.cb_dp_solve.argtypes = [c_void_p, c_void_p, c_double, P32, POINTER(DPResult)]
        L.cb_patterns_destroy.argtypes = [c_void_p]
        L.cb_matches_destroy.argtypes = [c_void_p]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(f"libcollage_b200 error {rc}: {lib().cb_last_error().decode()}")


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(POINTER(t))


def optimize_on_b200(g, registry, measurer, epsilon: float):
    """(kernels, cost_ms) of the op-level placement of the reference graph
    `g`; kernels are (pattern registration index, root id, sorted node ids)
    in the DP's pop order of their roots."""
    from paper_2111_00655_b200 import graph as cb_graph
    from paper_2111_00655_b200._encode import OP_KINDS
    from paper_2111_00655_b200.patterns import CompiledPatterns, parse_pattern
    L = lib()
    # 1. graph -> cb_graph (the JSON round trip keeps ids, attrs and shapes)
    from tensorplace.graph import Subgraph, graph_to_json
    cg = cb_graph.graph_from_json(json.loads(json.dumps(graph_to_json(g))))
    # 2. registry -> cb_patterns: pre-order position tables, backend per pattern
    backends = list(registry.backends)
    pats = list(registry.patterns)
    comp = CompiledPatterns([parse_pattern(bp.text()) for bp in pats],
                            [backends.index(bp.backend) for bp in pats])
    n_kinds = len(OP_KINDS)
    order = np.argsort(comp.root_kind, kind="stable").astype(np.int32)
    counts = np.bincount(comp.root_kind, minlength=n_kinds)
    kind_pat_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    hp = c_void_p()
    _check(L.cb_patterns_create(
        comp.n_pat, n_kinds, _p(comp.pos_ptr, c_int32), _p(comp.kind, c_int32),
        _p(comp.nargs, c_int32), _p(comp.parent, c_int32), _p(comp.argidx, c_int32),
        _p(comp.sid, c_int32), _p(comp.con_ptr, c_int32), _p(comp.con_key, c_int32),
        _p(comp.con_op, c_int8), _p(comp.con_val_ptr, c_int32), _p(comp.val_tag, c_int8),
        _p(comp.val_ival, c_int64), _p(comp.val_fval, c_double), _p(comp.con_lo, c_int64),
        _p(comp.con_hi, c_int64), _p(comp.backend, c_int32), _p(kind_pat_ptr, c_int32),
        _p(order, c_int32), byref(hp)))
    hm = c_void_p()
    try:
        # 3. every candidate match (candidates_at of every node), grouped by root
        _check(L.cb_match_all(cg.native, hp, byref(hm)))
        ng, nm, nmem, nb = (c_int64() for _ in range(4))
        _check(L.cb_matches_counts(hm, byref(ng), byref(nm), byref(nmem), byref(nb)))
        group_ptr = np.empty(ng.value + 1, np.int32)
        pat, root = np.empty(nm.value, np.int32), np.empty(nm.value, np.int32)
        mem_ptr, members = np.empty(nm.value + 1, np.int32), np.empty(nmem.value, np.int32)
        bind_ptr, binds = np.empty(nm.value + 1, np.int32), np.empty(max(nb.value, 1), np.int32)
        _check(L.cb_matches_download(hm, _p(group_ptr, c_int32), _p(pat, c_int32),
                                     _p(root, c_int32), _p(mem_ptr, c_int32),
                                     _p(members, c_int32), _p(bind_ptr, c_int32),
                                     _p(binds, c_int32)))
        ids = np.asarray(sorted(g.nodes), dtype=np.int64)  # node index -> id (ids ascending)
        # 4. kernel costs from the reference's own measurer
        costs = np.empty(nm.value)
        for m in range(nm.value):
            nodes = frozenset(int(ids[v]) for v in members[mem_ptr[m]:mem_ptr[m + 1]])
            costs[m] = measurer.measure_kernel(pats[pat[m]].backend, Subgraph(g, nodes))
        _check(L.cb_matches_set_costs(hm, _p(costs, c_double)))
        # 5. the DP
        kern = np.empty(len(g.nodes), np.int32)
        res = DPResult()
        _check(L.cb_dp_solve(cg.native, hm, float(epsilon), _p(kern, c_int32),
                             byref(res)))
        if not res.feasible:
            raise RuntimeError("no full placement")
        out = []
        for m in kern[:res.n_kernels].tolist():
            nodes = tuple(sorted(int(ids[v]) for v in members[mem_ptr[m]:mem_ptr[m + 1]]))
            out.append((int(pat[m]), int(ids[root[m]]), nodes))
        return out, res.cost_ms
    finally:
        if hm.value:
            L.cb_matches_destroy(hm)
        L.cb_patterns_destroy(hp)

