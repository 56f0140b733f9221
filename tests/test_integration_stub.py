"""INTEGRATION.md's reference-side binding (examples/tensorplace_b200.py):
raw ctypes calls into libcollage_b200.so from `tensorplace` objects give the
placement `optimize` gives.  Where the reference package is not importable
(the GPU box), `tensorplace` is this package -- the same API."""

from __future__ import annotations

import importlib
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _tensorplace():
    try:
        return importlib.import_module("tensorplace")
    except ImportError:
        import paper_2111_00655_b200 as pkg
        sys.modules["tensorplace"] = pkg
        for m in ("graph", "cost", "dp", "registry", "patterns"):
            sys.modules["tensorplace." + m] = importlib.import_module("paper_2111_00655_b200." + m)
        return pkg


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["resnet50", "bert_base", "nasrnn"])
def test_stub_matches_optimize(name, gpu):
    _tensorplace()
    sys.path.insert(0, os.path.join(ROOT, "examples"))
    import tensorplace_b200 as stub
    import paper_2111_00655_b200 as tp
    from paper_2111_00655_b200 import workloads
    g = workloads.CONFIGS[name]()
    bs = workloads.paper_backends(g, verify=False)
    kernels, cost = stub.optimize_on_b200(g, bs.registry, tp.SimMeasurer(bs.measurer.profiles), 0.01)
    res = tp.optimize(g, bs.registry, tp.SimMeasurer(bs.measurer.profiles), 0.01)
    assert cost == res.cost_ms
    got = sorted((k[0], k[1], k[2]) for k in kernels)
    want = sorted((a.backend_pattern.order, a.root, tuple(sorted(a.nodes)))
                  for a in res.placement.assignments)
    assert got == want
