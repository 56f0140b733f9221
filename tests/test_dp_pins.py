"""DP placements pinned on every BASELINE.json config.

The reference DP (tensorplace/dp.py:71-179) only finishes ResNet-50 and
BERT-base; for NasNet-A, the 10-step NasRNN and the 100k-node random DAG it
raises SearchLimitError.  The pins (tests/golden/dp_pins.json, written by
tests/golden/make_dp_pins.py) come from the oracle's second, independent
exact solver `or_dp_subtree`.  CPU tests below establish that solver:

* it returns the reference's own cost and kernels on every golden DP case
  (tests/test_oracle_golden.py runs it next to the covered-set restatement);
* it equals the covered-set restatement (or_dp, the reference's Algorithm 1
  in C) beyond the reference's state cap, on the golden cases the reference
  gave up on and on random DAGs with many parallel branches;
* the committed cases and pins are reproducible from the workload builders.

The GPU tests then require the device DP to return exactly the pinned
placement (cost, kernel list digest) on all five configs, with the
rounding window certified safe, and the random 100k DAG's fitness to match
the oracle on 256+ genomes.
"""

import gzip
import hashlib
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
from oracle import OracleCase, window_safe

CONFIGS = ["resnet50", "bert_base", "nasnet_a", "nasrnn", "random100k"]


def _pins():
    with open(os.path.join(GOLDEN, "dp_pins.json")) as fh:
        return json.load(fh)


def _case(name):
    with gzip.open(os.path.join(GOLDEN, "cases", f"{name}.json.gz"), "rt") as fh:
        return json.load(fh)


def _digest(obj):
    return hashlib.sha256(json.dumps(obj, separators=(",", ":")).encode()).hexdigest()


def _check_partition(oc, kernels, cost):
    """kernels cover every node once, each is a candidate match, and the
    cost is the reference's canonical total of them (fsum of cost + eps)."""
    seen = np.zeros(oc.n, np.int64)
    terms = []
    mt = oc._mt
    for order, root, nodes in kernels:
        v = oc.index[root]
        hit = [m for m in range(mt["group_ptr"][v], mt["group_ptr"][v + 1])
               if int(mt["pat"][m]) == order and
               sorted(oc.ids[x] for x in mt["members"][mt["mem_ptr"][m]:mt["mem_ptr"][m + 1]]) == nodes]
        assert len(hit) == 1
        terms += [float(oc.cost[hit[0]]), oc.epsilon]
        for nid in nodes:
            seen[oc.index[nid]] += 1
    assert np.all(seen == 1)
    assert math.fsum(terms) == cost


def test_subtree_solver_beyond_reference_cap():
    """dp_large cases the reference gave up on (20-38 nodes): the covered-set
    restatement with a 5 M-state budget finishes five of them and must agree;
    every result is a valid partition priced as the reference prices it."""
    agreed = 0
    for case in golden("dp_large"):
        if case["dp"].get("error") != "SearchLimitError":
            continue
        oc = OracleCase(case)
        oc.price()
        status, cost, kernels, regret = oc.dp_subtree()
        assert status == "ok" and window_safe(cost, regret)
        _check_partition(oc, kernels, cost)
        if len(case["graph"]["nodes"]) <= 30:
            s2, c2, k2 = oc.dp(max_states=5_000_000)
            if s2 == "ok":
                assert (c2, k2) == (cost, kernels), case["name"]
                agreed += 1
    assert agreed >= 5


def _random_case(seed):
    import random
    from paper_2111_00655_b200 import workloads
    from paper_2111_00655_b200.cost import profile_to_json
    from paper_2111_00655_b200.graph import graph_to_json
    rng = random.Random(seed)
    n = rng.randrange(8, 22)
    g = workloads.random_dag(n, seed=seed, ops=workloads.RANDOM_OPS[:rng.choice((3, 4, 6))],
                             window=rng.choice((None, 4, 8)))
    bs = workloads.random_backends(g, n_backends=rng.choice((2, 3, 4)), n_graph=1, seed=seed,
                                   fused_per_backend=rng.choice((2, 6, 10)))
    return json.loads(json.dumps({
        "graph": graph_to_json(g), "epsilon": rng.choice((0.01, 0.0, 0.5)),
        "backends": [[b.id, b.kind.value] for b in bs.registry.backends.values()],
        "patterns": [[bp.backend, bp.text(), bp.source.value] for bp in bs.registry.patterns],
        "profiles": {b: profile_to_json(p) for b, p in bs.measurer.profiles.items()}}))


def test_subtree_solver_equals_covered_set_on_random_dags():
    """150 random DAGs (8-21 nodes, several fused patterns per backend,
    ties from shared cost values, epsilon 0 included): the two oracle
    solvers agree on status, cost and kernels whenever the covered-set DP
    finishes and the rounding window is certified."""
    compared = 0
    for seed in range(150):
        case = _random_case(seed)
        oc = OracleCase(case)
        oc.price()
        s1, c1, k1, reg = oc.dp_subtree()
        s2, c2, k2 = oc.dp(max_states=2_000_000)
        if s2 == "limit":
            continue
        assert s1 == s2, seed
        if s1 == "ok" and window_safe(c1, reg):
            assert (c1, k1) == (c2, k2), seed
            compared += 1
    assert compared >= 100


def test_pins_are_reproducible():
    """The committed cases are what the workload builders produce today, and
    the independent solver still returns the pinned placement."""
    import sys
    sys.path.insert(0, GOLDEN)
    from make_dp_pins import case_of
    pins = _pins()
    assert sorted(pins) == sorted(CONFIGS)
    for name in CONFIGS:
        case = _case(name)
        pin = pins[name]
        assert _digest(case) == pin["case_sha256"], name
        if name != "random100k":  # 4 s to rebuild; its digest above pins the file
            assert _digest(case_of(name)) == pin["case_sha256"], name
        oc = OracleCase(case)
        oc.price()
        status, cost, kernels, regret = oc.dp_subtree()
        assert status == "ok" and cost == pin["cost"] and len(kernels) == pin["n_kernels"]
        assert _digest(kernels) == pin["kernels_sha256"], name
        assert window_safe(cost, regret) and pin["window_safe"]
        if name != "random100k":
            _check_partition(oc, kernels, cost)


# ------------------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name", CONFIGS)
def test_device_dp_matches_pin(gpu, name):
    """The device DP returns the pinned placement on every config: identical
    cost, identical canonical kernel list, rounding window certified."""
    import paper_2111_00655_b200 as tp
    from conftest import kernels_of
    from paper_2111_00655_b200 import workloads
    pin = _pins()[name]
    g = workloads.CONFIGS[name]()
    bs = workloads.random_backends(g, n_backends=8, n_graph=1, seed=0) if name == "random100k" \
        else workloads.paper_backends(g)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
    kernels = kernels_of(res.placement)
    assert res.cost_ms == pin["cost"]
    assert len(kernels) == pin["n_kernels"]
    if "kernels" in pin:
        assert kernels == pin["kernels"]
    assert _digest(kernels) == pin["kernels_sha256"]
    assert res.device["rounding_window_safe"]


@pytest.mark.gpu
def test_random100k_fitness_matches_oracle(gpu):
    """The config-5 fitness kernel (anchor walk) at full size against the
    oracle's restatement of the reference's graph-level pricing: 320 genomes
    of 99 446 bits at densities 0.02 / 0.5 / 0.98 and ES-bred rows."""
    import paper_2111_00655_b200 as tp
    from paper_2111_00655_b200 import workloads
    from paper_2111_00655_b200.es_device import DeviceEvolution
    pin = _pins()["random100k"]
    g = workloads.CONFIGS["random100k"]()
    bs = workloads.random_backends(g, n_backends=8, n_graph=1, seed=0)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
    plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                          res.kernel_matches)
    rng = np.random.default_rng(5)
    rows = [(rng.random((64, plan.k)) < d).astype(np.uint8) for d in (0.02, 0.5, 0.98)]
    bits = np.concatenate(rows)
    words = plan.words
    buf = np.zeros((len(bits), words * 8), np.uint8)
    pk = np.packbits(bits, axis=1, bitorder="little")
    buf[:, :pk.shape[1]] = pk
    packed = buf.view(np.uint64)
    # ES-bred rows: a few device generations from a random population
    es = DeviceEvolution(plan, 4096, seed=3)
    es.initialize()
    for _ in range(3):
        es.step()
    bred = es.pop[es.cur][:128].cpu().numpy().view(np.uint64)
    packed = np.concatenate([packed, bred])
    got = plan.evaluate_packed(np.ascontiguousarray(packed), np.empty(len(packed)))
    oc = OracleCase(_case("random100k"))
    oc.price()
    kernels = [[a.backend_pattern.order, a.root, sorted(a.nodes)] for a in res.placement.assignments]
    assert _digest(kernels) == pin["kernels_sha256"]
    want = oc.fitness(kernels, bs.graph_backend, packed, threads=os.cpu_count() or 1)
    assert plan.kernel_name() == "fitness_anchor_kernel"
    assert np.array_equal(got, want)
