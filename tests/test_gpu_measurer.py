"""Measurer cache protocol of device pricing against the reference
(tests/golden/measurer.json): the reference's DP calls
SimMeasurer.measure_kernel once per candidate (tensorplace/cost.py:248-263),
so a cold optimize fills the cache with one entry per distinct kernel key and
a warm rerun is pure lookup (acceptance test 07).  The device prices every
candidate in one launch; the cache and counters it leaves must be the same."""

import hashlib
import json
import math

import pytest

import paper_2111_00655_b200 as tp
from conftest import build_case, golden

pytestmark = pytest.mark.gpu

BY_NAME = {}
for s in ("fixtures", "models", "dp_random", "dp_ties"):
    for c in golden(s):
        BY_NAME[(s, c["name"])] = c
CASES = golden("measurer")


@pytest.mark.parametrize("want", CASES, ids=[c["name"] for c in CASES])
def test_cold_and_warm_runs_match_reference(gpu, want):
    case = BY_NAME[(want["suite"], want["name"])]
    g, reg, meas = build_case(case)
    runs = []
    for _ in range(2):
        reg._tables.clear()  # a fresh match table each run, as the reference re-matches
        res = tp.optimize(g, reg, meas, case["epsilon"])
        runs.append({"measure_calls": res.stats.measure_calls, "cache_hits": res.stats.cache_hits,
                     "computations": res.stats.computations})
        if len(runs) == 1:
            items = sorted(meas.cache.items())
    assert runs == want["runs"]
    assert len(items) == want["cache_size"]
    assert hashlib.sha256(json.dumps(items).encode()).hexdigest() == want["cache_sha256"]
    assert {"calls": meas.calls, "cache_hits": meas.cache_hits,
            "computations": meas.computations} == want["counters"]


def test_cached_costs_override_device_prices(gpu, tmp_path):
    """A cache loaded from disk (e.g. measured costs) wins over the profile,
    as in the reference; saving and reloading round-trips."""
    case = golden("fixtures")[0]
    g, reg, meas = build_case(case)
    res = tp.optimize(g, reg, meas, case["epsilon"])
    path = tmp_path / "costs.jsonl"
    tp.cache_save(meas.cache, str(path))
    cache = tp.cache_load(str(path))
    for key, _ in list(cache.items()):
        cache.put(key, 1.0)  # every kernel now costs 1 ms
    g2, reg2, _ = build_case(case)
    meas2 = tp.SimMeasurer(meas.profiles, cache)
    res2 = tp.optimize(g2, reg2, meas2, case["epsilon"])
    assert res2.stats.computations == 0
    n = len(res2.placement)
    assert res2.cost_ms == math.fsum([1.0, case["epsilon"]] * n)
    assert res.cost_ms != res2.cost_ms
