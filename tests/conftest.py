"""Shared fixtures.  `-m gpu` tests need a CUDA device and the built
libcollage_b200.so; everything else runs on CPU (oracle, host logic, ABI)."""

from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the native library")


def golden(name: str) -> list:
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        return json.load(fh)


def build_case(case: dict):
    """(graph, registry, measurer) of this package for a golden case."""
    import paper_2111_00655_b200 as tp
    from paper_2111_00655_b200.cost import profile_from_json
    g = tp.graph_from_json(case["graph"])
    reg = tp.PatternRegistry()
    for bid, kind in case["backends"]:
        reg.add_backend(tp.BackendDescriptor(bid, tp.BackendKind(kind)))
    for bid, text, source in case["patterns"]:
        assert reg.add_pattern(bid, text, tp.PatternSource(source))
    meas = tp.SimMeasurer({b: profile_from_json(d) for b, d in case["profiles"].items()})
    return g, reg, meas


def kernels_of(placement) -> list:
    return [[a.backend_pattern.order, a.root, sorted(a.nodes)] for a in placement.assignments]


@pytest.fixture(scope="session")
def gpu():
    from paper_2111_00655_b200 import _native as nat
    if not nat.device_available():
        pytest.fail("GPU test selected but no CUDA device / native library is available")
    return True
