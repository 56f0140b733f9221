"""libcollage_b200.so: loads without a GPU, exports the declared C ABI, and
its host-side pieces (exact summation, graph analysis) are right."""

import ctypes
import math
import os
import random
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2111_00655_b200 import _native as nat


def _declared():
    with open(os.path.join(ROOT, "include", "collage_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(cb_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported_and_bound():
    lib = nat.lib()
    declared = _declared()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(nat.EXPORTED_SYMBOLS)
    assert lib.cb_abi_version() == 1


def test_device_entry_points_fail_loudly_without_a_gpu():
    if nat.device_available():
        pytest.skip("a GPU is present")
    import paper_2111_00655_b200 as tp
    g = tp.ComputationGraph([tp.GraphInput("x", (4,))],
                            [tp.OperatorNode(0, "relu", {}, (tp.InputRef("x"),), (4,))], [0])
    with pytest.raises(nat.DeviceUnavailableError):
        tp.match_at(g, 0, tp.parse_pattern("relu(*)"))


def _fx_sum(xs):
    a = np.asarray(xs, dtype=np.float64)
    out = ctypes.c_double()
    exact = ctypes.c_int32()
    nat.check(nat.lib().cb_fx_sum(nat.ptr(a, ctypes.c_double), len(a), ctypes.byref(out),
                                  ctypes.byref(exact)))
    return out.value, exact.value


def test_fixed_point_sum_equals_fsum():
    rng = random.Random(5)
    for _ in range(300):
        xs = [rng.random() * 10 ** rng.randint(-20, 15) for _ in range(rng.randint(0, 60))]
        got, exact = _fx_sum(xs)
        assert exact == 1
        assert got == math.fsum(xs)
    # halfway cases round to even exactly like fsum
    for xs in ([1.0, 2.0 ** -53], [1.0, 2.0 ** -53, 2.0 ** -105], [3.0, 2.0 ** -52],
               [0.1, 0.2, 0.3], [1e-19, 1.0, -0.0]):
        assert _fx_sum(xs)[0] == math.fsum(xs)


def test_fixed_point_range_is_reported():
    assert _fx_sum([2.0 ** -100])[1] == 1  # a power of two keeps no low bits
    assert _fx_sum([2.0 ** -100 * (1 + 2.0 ** -52)])[1] == 0  # bit below 2^-128 lost
    assert _fx_sum([2.0 ** 70])[1] == 0    # above 2^64
    assert _fx_sum([-1.0])[1] == 0


def _brute_pdom(g, v):
    paths, acc = [], []

    def walk(n):
        acc.append(n)
        if n in g.outputs:
            paths.append(set(acc))
        for c in g.consumers(n):
            walk(c)
        acc.pop()

    walk(v)
    common = set(paths[0])
    for p in paths[1:]:
        common &= p
    return common


def test_graph_analysis_matches_definitions():
    from paper_2111_00655_b200 import workloads
    for seed in range(40):
        g = workloads.random_dag(random.Random(seed).randint(2, 14), seed=seed)
        order = g.topo_order()
        pos = {v: i for i, v in enumerate(order)}
        for v in g.nodes:
            for p in g.node_predecessors(v):
                assert pos[p] < pos[v]
                assert g.depth(v) > g.depth(p)
        for v in g.nodes:
            pd = _brute_pdom(g, v)
            for d in g.nodes:
                assert g.post_dominates(d, v) == (d in pd)
            strict = pd - {v}
            ip = g.post_dominator(v)
            if not strict:
                assert ip is None
            else:
                assert ip == min(strict, key=pos.__getitem__)
