"""ctypes front end of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product
package.  `OracleCase` encodes a golden case (graph JSON, backends,
patterns, profiles) with its own encoder and runs the restated reference
algorithms: matcher, kernel pricing, the covered-set DP and the graph-level
fitness of offload genomes.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_int8, c_int32, c_int64, c_uint8, c_uint64

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = ctypes.CDLL(LIB)
        P32 = POINTER(c_int32)
        _lib.or_match_all.restype = c_int
        _lib.or_match_all.argtypes = [c_int, P32, P32, P32, POINTER(c_uint8), P32, P32,
                                      POINTER(c_int8), POINTER(c_int64), POINTER(c_double),
                                      c_int, P32, P32, P32, P32, P32, P32, P32, P32,
                                      POINTER(c_int8), P32, POINTER(c_int8), POINTER(c_int64),
                                      POINTER(c_double), POINTER(c_int64), POINTER(c_int64),
                                      c_int, P32, P32] + [POINTER(P32)] * 6 + [P32]
        _lib.or_free.argtypes = [ctypes.c_void_p]
        _lib.or_price.restype = c_int
        _lib.or_price.argtypes = [c_int, P32, P32, P32, P32, P32, POINTER(c_double), c_int,
                                  POINTER(c_double), POINTER(c_double), POINTER(c_uint8),
                                  POINTER(c_uint8), c_int, POINTER(c_double),
                                  POINTER(c_double), POINTER(c_int8)]
        _lib.or_dp.restype = c_int
        _lib.or_dp.argtypes = [c_int, P32, P32, P32, POINTER(c_uint8), c_int, P32, P32, P32, P32,
                               POINTER(c_double), c_double, c_int, P32, P32, POINTER(c_double),
                               POINTER(c_int64), P32, P32]
        _lib.or_dp_subtree.restype = c_int
        _lib.or_dp_subtree.argtypes = [c_int, P32, P32, P32, POINTER(c_uint8), c_int, P32, P32, P32,
                                       P32, POINTER(c_double), c_double, c_int64, P32, P32,
                                       POINTER(c_double), POINTER(c_double), P32, POINTER(c_int64)]
        _lib.or_fitness.restype = c_int
        _lib.or_fitness.argtypes = [c_int, P32, P32, P32, P32, P32, P32, POINTER(c_double), c_int,
                                    P32, c_int, POINTER(c_uint8), POINTER(c_double),
                                    POINTER(c_double), c_int, c_double, POINTER(c_uint64),
                                    c_int64, c_int, c_int, POINTER(c_double)]
    return _lib


def window_safe(cost: float, min_regret: float | None) -> bool:
    """True when no rounded comparison of the reference can disagree with the
    exact one: any two states of one cover differ by a sum of decision
    regrets, so a difference of at least 4 ulp(cost) (states cost at most
    twice the total before they differ by more than the total) keeps their
    rounded costs apart."""
    import math
    if min_regret is None or math.isinf(min_regret):
        return True
    return min_regret >= 4 * math.ulp(cost)


def _p(a, t):
    return a.ctypes.data_as(POINTER(t))


def _i32(x):
    return np.ascontiguousarray(x, dtype=np.int32)


class OracleCase:
    """A golden case encoded for the oracle."""

    def __init__(self, case: dict):
        from paper_2111_00655_b200._encode import ATTR_KEYS, OP_KINDS, encode_value
        from paper_2111_00655_b200.patterns import CompiledPatterns, parse_pattern
        doc = case["graph"]
        nodes = sorted(doc["nodes"], key=lambda n: n["id"])
        self.ids = [n["id"] for n in nodes]
        index = {nid: i for i, nid in enumerate(self.ids)}
        self.index = index
        n = len(nodes)
        self.n = n
        self.kind = _i32([OP_KINDS(nd["op"]) for nd in nodes])
        src, ptr = [], [0]
        akey, atag, aival, afval, aptr = [], [], [], [], [0]
        vol = []
        for nd in nodes:
            for r in nd["inputs"]:
                src.append(-1 if isinstance(r, dict) else index[r])
            ptr.append(len(src))
            for k in sorted(nd.get("attrs", {})):
                t, iv, fv = encode_value(nd["attrs"][k])
                akey.append(ATTR_KEYS(k)); atag.append(t); aival.append(iv); afval.append(fv)
            aptr.append(len(akey))
            v = 1
            for d in nd["shape"]:
                v *= d
            vol.append(float(v))
        self.in_ptr, self.in_src = _i32(ptr), _i32(src)
        self.is_output = np.zeros(n, np.uint8)
        for o in doc["outputs"]:
            self.is_output[index[o]] = 1
        self.attr_ptr, self.attr_key = _i32(aptr), _i32(akey)
        self.attr_tag = np.asarray(atag, np.int8)
        self.attr_ival = np.asarray(aival, np.int64)
        self.attr_fval = np.asarray(afval, np.float64)
        self.volume = np.asarray(vol, np.float64)
        self.backends = [b for b, _ in case.get("backends", [])]
        self.backend_kind = {b: k for b, k in case.get("backends", [])}
        pats = [p for p in case.get("patterns", []) if not isinstance(p, str)]
        self.pattern_backend = [self.backends.index(b) for b, _, _ in pats]
        self.patterns = [parse_pattern(t) for _, t, _ in pats]
        self.compiled = CompiledPatterns(self.patterns, self.pattern_backend)
        self.profiles = case.get("profiles", {})
        self.epsilon = case.get("epsilon", 0.01)
        self._mt = None

    # -- matcher -------------------------------------------------------------------
    def match_all(self, compiled=None):
        from paper_2111_00655_b200._encode import OP_KINDS
        c = compiled or self.compiled
        n_kinds = len(OP_KINDS)
        order = np.argsort(c.root_kind, kind="stable") if c.n_pat else np.zeros(0, np.int64)
        kind_pat = _i32(order)
        counts = np.bincount(c.root_kind, minlength=n_kinds) if c.n_pat else np.zeros(n_kinds)
        kptr = _i32(np.concatenate([[0], np.cumsum(counts)]))
        outs = [POINTER(c_int32)() for _ in range(6)]
        nm = c_int32()
        L = lib()
        rc = L.or_match_all(
            self.n, _p(self.kind, c_int32), _p(self.in_ptr, c_int32), _p(self.in_src, c_int32),
            _p(self.is_output, c_uint8), _p(self.attr_ptr, c_int32), _p(self.attr_key, c_int32),
            _p(self.attr_tag, c_int8), _p(self.attr_ival, c_int64), _p(self.attr_fval, c_double),
            c.n_pat, _p(c.pos_ptr, c_int32), _p(c.kind, c_int32), _p(c.nargs, c_int32),
            _p(c.parent, c_int32), _p(c.argidx, c_int32), _p(c.sid, c_int32),
            _p(c.con_ptr, c_int32), _p(c.con_key, c_int32), _p(c.con_op, c_int8),
            _p(c.con_val_ptr, c_int32), _p(c.val_tag, c_int8), _p(c.val_ival, c_int64),
            _p(c.val_fval, c_double), _p(c.con_lo, c_int64), _p(c.con_hi, c_int64), n_kinds,
            _p(kptr, c_int32), _p(kind_pat, c_int32), *[ctypes.byref(o) for o in outs],
            ctypes.byref(nm))
        assert rc == 0, "oracle: graph has a cycle"
        m = nm.value
        sizes = {"group_ptr": self.n + 1, "pat": m, "mem_ptr": m + 1}
        res = {}
        names = ["group_ptr", "pat", "mem_ptr", "members", "bind_ptr", "binds"]
        for name, o in zip(names, outs):
            if name in sizes:
                cnt = sizes[name]
            elif name == "members":
                cnt = res["mem_ptr"][-1]
            elif name == "bind_ptr":
                cnt = m + 1
            else:
                cnt = res["bind_ptr"][-1]
            res[name] = np.ctypeslib.as_array(o, shape=(int(cnt),)).copy() if cnt else \
                np.zeros(0, np.int32)
            L.or_free(ctypes.cast(o, ctypes.c_void_p))
        res["backend"] = _i32([c.backend[p] for p in res["pat"]])
        res["n"] = m
        if compiled is None:
            self._mt = res
        return res

    def candidates(self) -> dict:
        """{node id: [(pattern index, sorted node ids, binding)]} as the golden stores it."""
        mt = self._mt or self.match_all()
        out = {}
        for v in range(self.n):
            rows = []
            for m in range(mt["group_ptr"][v], mt["group_ptr"][v + 1]):
                pat = int(mt["pat"][m])
                mem = sorted(self.ids[x] for x in mt["members"][mt["mem_ptr"][m]:mt["mem_ptr"][m + 1]])
                binds = mt["binds"][mt["bind_ptr"][m]:mt["bind_ptr"][m + 1]]
                paths = self.compiled.paths[pat]
                binding = sorted((list(paths[i]), self.ids[x]) for i, x in enumerate(binds))
                rows.append([pat, mem, [[p, x] for p, x in binding]])
            out[str(self.ids[v])] = rows
        return out

    # -- pricing -------------------------------------------------------------------
    def price(self):
        from paper_2111_00655_b200._encode import OP_KINDS
        mt = self._mt or self.match_all()
        n_kinds = len(OP_KINDS)
        nb = len(self.backends)
        coeff = np.zeros((nb, n_kinds)); over = np.zeros((nb, n_kinds))
        has = np.zeros((nb, n_kinds), np.uint8); has_prof = np.zeros(nb, np.uint8)
        sizes = np.diff(mt["mem_ptr"]) if mt["n"] else np.ones(1, np.int64)
        stride = int(sizes.max()) + 1
        pw = np.ones((nb, stride))
        for b, bid in enumerate(self.backends):
            prof = self.profiles.get(bid)
            if prof is None:
                continue
            has_prof[b] = 1
            for op, e in prof["ops"].items():
                k = OP_KINDS(op)
                if k < n_kinds:
                    coeff[b, k] = float(e["coeff"]); over[b, k] = float(e["overhead"]); has[b, k] = 1
            disc = float(prof.get("fusion_discount", 1.0))
            for e in range(stride):
                pw[b, e] = disc ** e
        cost = np.empty(mt["n"]); err = np.zeros(mt["n"], np.int8)
        lib().or_price(mt["n"], None, _p(mt["mem_ptr"], c_int32), _p(mt["members"], c_int32),
                       _p(mt["backend"], c_int32), _p(self.kind, c_int32),
                       _p(self.volume, c_double), n_kinds, _p(coeff, c_double),
                       _p(over, c_double), _p(has, c_uint8), _p(has_prof, c_uint8), stride,
                       _p(pw, c_double), _p(cost, c_double), _p(err, c_int8))
        self.cost = cost
        return cost, err

    # -- DP ----------------------------------------------------------------------------
    def dp(self, max_states: int = 50_000):
        """(status, cost, kernels) with status 'ok' | 'uncoverable' | 'limit';
        kernels as [[pattern order, root id, sorted node ids]] canonical."""
        mt = self._mt or self.match_all()
        if not hasattr(self, "cost"):
            self.price()
        kern = np.empty(self.n + 1, np.int32)
        nk = c_int32(); cost = c_double(); relax = c_int64(); peak = c_int32(); fz = c_int32()
        rc = lib().or_dp(self.n, _p(self.kind, c_int32), _p(self.in_ptr, c_int32),
                         _p(self.in_src, c_int32), _p(self.is_output, c_uint8), mt["n"],
                         _p(mt["group_ptr"], c_int32), _p(mt["pat"], c_int32),
                         _p(mt["mem_ptr"], c_int32), _p(mt["members"], c_int32),
                         _p(self.cost, c_double), float(self.epsilon), int(max_states),
                         _p(kern, c_int32), ctypes.byref(nk), ctypes.byref(cost),
                         ctypes.byref(relax), ctypes.byref(peak), ctypes.byref(fz))
        self.dp_relaxations, self.dp_states = relax.value, peak.value
        self.first_zero = self.ids[fz.value] if fz.value >= 0 else None
        if rc == 1:
            return "uncoverable", None, None
        if rc == 2:
            return "limit", None, None
        ks = kern[:nk.value]
        return "ok", cost.value, self.kernels_json(ks)

    def dp_subtree(self, max_set_entries: int = 2_000_000_000):
        """The independent exact solver (or_dp_subtree): (status, cost,
        kernels, min_regret) with status 'ok' | 'uncoverable' | 'memory'.
        `window_safe(cost, min_regret)` tells whether the reference's rounded
        comparisons provably pick the same partition."""
        mt = self._mt or self.match_all()
        if not hasattr(self, "cost"):
            self.price()
        kern = np.empty(self.n + 1, np.int32)
        ipdom = np.empty(self.n + 1, np.int32)
        nk = c_int32(); cost = c_double(); reg = c_double(); ties = c_int64()
        rc = lib().or_dp_subtree(self.n, _p(self.kind, c_int32), _p(self.in_ptr, c_int32),
                                 _p(self.in_src, c_int32), _p(self.is_output, c_uint8), mt["n"],
                                 _p(mt["group_ptr"], c_int32), _p(mt["pat"], c_int32),
                                 _p(mt["mem_ptr"], c_int32), _p(mt["members"], c_int32),
                                 _p(self.cost, c_double), float(self.epsilon),
                                 int(max_set_entries), _p(kern, c_int32), ctypes.byref(nk),
                                 ctypes.byref(cost), ctypes.byref(reg), _p(ipdom, c_int32),
                                 ctypes.byref(ties))
        self.subtree_ties = ties.value
        if rc == 1:
            return "uncoverable", None, None, None
        if rc == 4:
            return "memory", None, None, None
        assert rc == 0, rc
        self.ipdom = ipdom[:self.n].copy()
        return "ok", cost.value, self.kernels_json(kern[:nk.value]), reg.value

    def kernels_json(self, matches) -> list:
        mt = self._mt
        rows = []
        for m in matches:
            mem = sorted(self.ids[x] for x in mt["members"][mt["mem_ptr"][m]:mt["mem_ptr"][m + 1]])
            root = self.ids[int(np.searchsorted(mt["group_ptr"], m, side="right") - 1)]
            rows.append([int(mt["pat"][m]), root, mem])
        rows.sort(key=lambda r: r[2])
        return rows

    def match_ids(self, kernels_json) -> np.ndarray:
        """Match index of [[order, root, nodes]] kernels (canonical order kept)."""
        mt = self._mt or self.match_all()
        out = []
        for order, root, nodes in kernels_json:
            v = self.index[root]
            hit = [m for m in range(mt["group_ptr"][v], mt["group_ptr"][v + 1])
                   if int(mt["pat"][m]) == order]
            out.append(hit[0])
        return _i32(out)

    # -- fitness -------------------------------------------------------------------------
    def fitness(self, kernels_json, target: str, genomes, threads: int = 1) -> np.ndarray:
        mt = self._mt or self.match_all()
        if not hasattr(self, "cost"):
            self.price()
        km = self.match_ids(kernels_json)
        nb = len(self.backends)
        is_graph = np.asarray([self.backend_kind[b] == "graph_inference_library"
                               for b in self.backends], np.uint8)
        alpha = np.zeros(nb); floor = np.ones(nb)
        for b, bid in enumerate(self.backends):
            prof = self.profiles.get(bid, {})
            alpha[b] = float(prof.get("region_alpha", 0.05))
            floor[b] = float(prof.get("region_floor", 0.7))
        if isinstance(genomes, np.ndarray) and genomes.dtype == np.uint64:
            packed = np.ascontiguousarray(genomes)
        else:
            g = np.asarray(genomes, np.uint8)
            k = g.shape[1] if g.ndim == 2 else 0
            words = max(1, (k + 63) // 64)
            buf = np.zeros((len(g), words * 8), np.uint8)
            if k:
                pk = np.packbits(g, axis=1, bitorder="little")
                buf[:, :pk.shape[1]] = pk
            packed = buf.view(np.uint64)
        out = np.empty(packed.shape[0])
        lib().or_fitness(self.n, _p(self.in_ptr, c_int32), _p(self.in_src, c_int32),
                         _p(mt["group_ptr"], c_int32), _p(mt["mem_ptr"], c_int32),
                         _p(mt["members"], c_int32), _p(mt["backend"], c_int32),
                         _p(self.cost, c_double), len(km), _p(km, c_int32), nb,
                         _p(is_graph, c_uint8), _p(alpha, c_double), _p(floor, c_double),
                         self.backends.index(target), float(self.epsilon),
                         _p(packed, c_uint64), packed.shape[0], packed.shape[1], threads,
                         _p(out, c_double))
        return out
