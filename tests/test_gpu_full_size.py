"""Full-size configurations (BASELINE.json configs) checked through
size-independent properties, each against an independent code path:

* the DP's cost equals the additive cost of its placement recomputed on the
  host by `SimProfile.kernel_cost` + math.fsum (device pricing and the DP's
  exact accumulation vs Python floats);
* the placement validates (batched device re-match + host cover/acyclicity);
* every genome's GPU fitness equals the graph-level cost of its decoded
  placement priced by the native single-placement routine (union-find over
  kernels, no frontier program);
* NasRNN / NasNet-A exceed the reference's 50 000-state cap, so they are
  only checked this way (the CPU oracle cannot enumerate them either).
"""

import math

import numpy as np
import pytest

import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads

pytestmark = pytest.mark.gpu

CONFIGS = ["resnet50", "bert_base", "nasnet_a", "nasrnn"]


def _setup(name):
    g = workloads.CONFIGS[name]()
    bs = workloads.paper_backends(g)
    return g, bs


@pytest.mark.parametrize("name", CONFIGS)
def test_dp_cost_is_the_additive_cost_of_its_placement(gpu, name):
    g, bs = _setup(name)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01, validate=True)
    costs = [bs.measurer.profiles[a.backend_pattern.backend].kernel_cost(tp.Subgraph(g, a.nodes))
             for a in res.placement.assignments]
    assert res.cost_ms == math.fsum(costs + [0.01] * len(costs))
    assert res.device["rounding_window_safe"]
    assert sorted(v for a in res.placement.assignments for v in a.nodes) == sorted(g.nodes)


@pytest.mark.parametrize("name", CONFIGS)
def test_fitness_equals_single_placement_pricing(gpu, name):
    g, bs = _setup(name)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
    plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                          res.kernel_matches)
    rng = np.random.default_rng(11)
    genomes = rng.integers(0, 2, size=(40, plan.k), dtype=np.uint8)
    feasible = np.array([k != 0 for k in plan.rep_kind], dtype=np.uint8)
    genomes[20:] &= feasible  # half of them guaranteed feasible
    genomes[0] = 0
    fit = plan.evaluate(genomes)
    gb = bs.registry.graph_backend_ids()
    for bits, f in zip(genomes, fit):
        dec = plan.decode(bits.tolist(), res.placement)
        if dec is None:
            assert math.isinf(f)
            continue
        want = tp.placement_cost_graphlevel(bs.measurer, g, dec, 0.01, gb)
        assert f == want
    assert fit[0] == plan.seed_cost == tp.placement_cost_graphlevel(
        bs.measurer, g, res.placement, 0.01, gb)


def test_random_dag_100k_end_to_end(gpu):
    g = workloads.random_dag(100_000, seed=0, ops=workloads.RANDOM_OPS, window=64)
    bs = workloads.random_backends(g, n_backends=8, n_graph=1, seed=0)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
    assert len(res.placement) > 0
    cov = np.zeros(len(g.nodes), dtype=np.int64)
    for a in res.placement.assignments:
        for v in a.nodes:
            cov[v] += 1
    assert np.all(cov == 1)
    costs = [bs.measurer.profiles[a.backend_pattern.backend].kernel_cost(tp.Subgraph(g, a.nodes))
             for a in res.placement.assignments]
    assert res.cost_ms == math.fsum(costs + [0.01] * len(costs))
    plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                          res.kernel_matches)
    rng = np.random.default_rng(3)
    genomes = rng.integers(0, 2, size=(4, plan.k), dtype=np.uint8)
    fit = plan.evaluate(genomes)
    for bits, f in zip(genomes[:2], fit[:2]):
        dec = plan.decode(bits.tolist(), res.placement)
        want = math.inf if dec is None else tp.placement_cost_graphlevel(
            bs.measurer, g, dec, 0.01, bs.registry.graph_backend_ids())
        assert f == want


def test_nasrnn_cell_matches_oracle_beyond_reference_cap(gpu):
    """One NasRNN cell (47 nodes): the reference DP exceeds 200 000 states; the
    CPU oracle's covered-set DP solves it with a 30 M-state cap
    (tests/golden/make_oracle_large.py) and the device DP must return the
    identical placement and cost."""
    import json
    import os
    from conftest import GOLDEN, build_case, kernels_of
    with open(os.path.join(GOLDEN, "oracle_large.json")) as fh:
        cases = json.load(fh)
    for case in cases:
        g, reg, meas = build_case(case)
        res = tp.optimize(g, reg, meas, case["epsilon"])
        want = case["oracle_dp"]
        assert res.cost_ms == want["cost"], case["name"]
        assert kernels_of(res.placement) == want["kernels"], case["name"]


@pytest.mark.parametrize("name", CONFIGS)
def test_fitness_matches_oracle_at_full_size(gpu, name):
    """Every BASELINE model config at full size: the automatically chosen
    fitness kernel (the FSM walk for all four) against the CPU oracle's
    restatement of the reference's graph-level pricing, bit for bit, on
    sparse, random and dense genomes."""
    import json
    from oracle import OracleCase
    from paper_2111_00655_b200.cost import profile_to_json
    from paper_2111_00655_b200.graph import graph_to_json
    g, bs = _setup(name)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
    plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                          res.kernel_matches)
    rng = np.random.default_rng(21)
    feasible = np.array([k != 0 for k in plan.rep_kind], dtype=np.uint8)
    rows = [(rng.random((700, plan.k)) < d).astype(np.uint8) & feasible for d in (0.05, 0.5, 0.95)]
    rows.append((rng.random((100, plan.k)) < 0.5).astype(np.uint8))  # infeasible bits allowed
    genomes = np.concatenate(rows)
    case = json.loads(json.dumps({
        "graph": graph_to_json(g),
        "backends": [[b.id, b.kind.value] for b in bs.registry.backends.values()],
        "patterns": [[bp.backend, bp.text(), bp.source.value] for bp in bs.registry.patterns],
        "profiles": {b: profile_to_json(p) for b, p in bs.measurer.profiles.items()},
        "epsilon": 0.01}))
    oc = OracleCase(case)
    oc.price()
    kernels = [[a.backend_pattern.order, a.root, sorted(a.nodes)] for a in res.placement.assignments]
    want = oc.fitness(kernels, bs.graph_backend, genomes, threads=8)
    assert plan.kernel_name().startswith("fitness_fsm_kernel")
    assert np.array_equal(plan.evaluate(genomes), want)
