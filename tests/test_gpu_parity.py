"""GPU path (libcollage_b200 through the package API) against the reference's
golden outputs and the CPU oracle: bit-exact matches, placements and costs."""


import numpy as np
import pytest

import paper_2111_00655_b200 as tp
from conftest import build_case, golden, kernels_of
from oracle import OracleCase

pytestmark = pytest.mark.gpu

DP_SUITES = ["fixtures", "dp_random", "dp_ties", "dp_large", "es_random", "models"]


def _cases(suites, key=None):
    for s in suites:
        for c in golden(s):
            if key is None or key in c:
                yield pytest.param(c, id=c["name"])


@pytest.mark.parametrize("case", list(_cases(DP_SUITES, "candidates")))
def test_candidates_match_reference(gpu, case):
    g, reg, _ = build_case(case)
    for nid in sorted(g.nodes):
        got = [[bp.order, sorted(m.nodes.node_ids), [[list(p), v] for p, v in m.binding]]
               for bp, m in reg.candidates_at(g, nid)]
        assert got == case["candidates"][str(nid)], nid


def test_match_all_matches_reference(gpu):
    checked = 0
    for case in golden("matcher"):
        g = tp.graph_from_json(case["graph"])
        for text, want in case["matches"].items():
            got = [[m.root, sorted(m.nodes.node_ids), [[list(p), v] for p, v in m.binding]]
                   for m in tp.match_all(g, tp.parse_pattern(text))]
            assert got == want, (case["name"], text)
            for root, nodes, _ in want[:2]:
                m = tp.match_at(g, root, tp.parse_pattern(text))
                assert m is not None and sorted(m.nodes.node_ids) == nodes
            checked += 1
    assert checked >= 300


@pytest.mark.parametrize("case", list(_cases(DP_SUITES)))
def test_dp_matches_reference(gpu, case):
    g, reg, meas = build_case(case)
    exp = case["dp"]
    if exp.get("error") == "UncoverableGraphError":
        with pytest.raises(tp.UncoverableGraphError) as info:
            tp.optimize(g, reg, meas, case["epsilon"])
        if exp["node_ids"]:
            assert list(info.value.node_ids) == exp["node_ids"]
            assert list(info.value.op_kinds) == exp["op_kinds"]
        return
    res = tp.optimize(g, reg, meas, case["epsilon"])
    if exp.get("error") == "SearchLimitError":
        # the reference gave up; check against the oracle's independent exact
        # solver (equal to its covered-set DP wherever that finishes,
        # tests/test_dp_pins.py)
        oc = OracleCase({**case, "patterns": case["patterns"]})
        oc.price()
        status, cost, kernels, _ = oc.dp_subtree()
        assert status == "ok"
        assert res.cost_ms == cost
        assert kernels_of(res.placement) == kernels
        return
    assert res.cost_ms == exp["cost"]
    assert kernels_of(res.placement) == exp["kernels"]
    assert res.device["rounding_window_safe"]
    assert res.stats.candidates_total == sum(len(v) for v in case.get("candidates", {}).values()) \
        or "candidates" not in case


@pytest.mark.parametrize("case", list(_cases(DP_SUITES, "es")))
def test_fitness_matches_reference(gpu, case):
    g, reg, meas = build_case(case)
    res = tp.optimize(g, reg, meas, case["epsilon"])
    es = case["es"]
    plan = tp.FitnessPlan(g, reg, meas, res.placement, case["epsilon"], es["graph_backend"],
                          res.kernel_matches)
    assert plan.k == es["genome_length"]
    fit = plan.evaluate(es["genomes"])
    assert np.array_equal(fit, np.array(es["fitness"]))
    assert plan.seed_cost == es["fitness"][0]


@pytest.mark.parametrize("case", list(_cases(DP_SUITES, "es")))
def test_evolve_matches_reference(gpu, case):
    g, reg, meas = build_case(case)
    ev = case["es"].get("evolve")
    if ev is None:
        pytest.skip("no evolve run recorded")
    res = tp.optimize(g, reg, meas, case["epsilon"])
    out = tp.evolve(g, reg, meas, res.placement, case["epsilon"], tp.ESConfig(**ev["config"]),
                    graph_backend=case["es"]["graph_backend"])
    assert [list(h) for h in out.history] == ev["history"]
    assert out.cost_ms == ev["cost"]
    assert out.seed_cost_ms == ev["seed_cost"]
    assert out.evaluations == ev["evaluations"]
    assert kernels_of(out.placement) == ev["kernels"]
    opt = case["es"].get("optimal_genome")
    if opt is not None:
        assert out.cost_ms >= opt["cost"]


@pytest.mark.parametrize("case", list(_cases(["rules"])))
def test_rule_generation_with_device_self_check(gpu, case):
    from paper_2111_00655_b200.rules import rule_from_json
    g = tp.graph_from_json(case["graph"])
    rule = rule_from_json(case["rule"])
    gen = tp.generate_patterns(rule, g)  # verify=True: every pattern re-matched on the GPU
    assert [[tp.pattern_to_text(x.pattern), x.origin, sorted(x.source_nodes)] for x in gen] \
        == case["generated"]


def test_decode_and_validate_on_device(gpu):
    case = golden("fixtures")[2]
    g, reg, meas = build_case(case)
    res = tp.optimize(g, reg, meas, 0.01)
    tp.validate_placement(g, res.placement)
    dec = tp.decode_genome(g, reg, res.placement, (0, 1, 1, 1, 0, 0), "simgraph")
    assert [a.backend_pattern.backend for a in dec.assignments] == \
        ["cpu", "simgraph", "simgraph", "simgraph", "cpu", "cpu"]
    assert tp.decode_genome(g, reg, res.placement, (1, 0, 0, 0, 0, 0), "simgraph") is None
    cost = tp.placement_cost_graphlevel(meas, g, dec, 0.01, reg.graph_backend_ids())
    assert cost == 5.794


def _plan_and_oracle(case):
    g, reg, meas = build_case(case)
    res = tp.optimize(g, reg, meas, case["epsilon"])
    target = case.get("es", {}).get("graph_backend") or reg.graph_backend_ids()[-1]
    plan = tp.FitnessPlan(g, reg, meas, res.placement, case["epsilon"], target,
                          res.kernel_matches)
    oc = OracleCase(case)
    oc.price()
    return res, plan, oc, target


@pytest.mark.parametrize("case", list(_cases(["models", "es_random"], "es"))[:30])
def test_fitness_paths_agree_with_oracle(gpu, case):
    res, plan, oc, target = _plan_and_oracle(case)
    rng = np.random.default_rng(7)
    genomes = rng.integers(0, 2, size=(3000, plan.k), dtype=np.uint8)
    # bias some rows towards long offloaded runs (large regions)
    genomes[:1000] |= rng.integers(0, 2, size=(1000, plan.k), dtype=np.uint8)
    genomes[1000:1500] = 1
    want = oc.fitness(kernels_of(res.placement), target, genomes)
    got_auto = plan.evaluate(genomes)
    assert np.array_equal(got_auto, want)
    plan.set_path("unionfind")
    assert np.array_equal(plan.evaluate(genomes), want)
    if plan.info.frontier_slots:
        for path in ("wide", "anchor"):
            plan.set_path(path)
            assert np.array_equal(plan.evaluate(genomes), want), path
        plan.set_pool(1)
        assert np.array_equal(plan.evaluate(genomes), want), "anchor, pool of 1"
        plan.set_pool(16)
    if 0 < plan.info.frontier_slots <= 32:
        for path in ("frontier", "frontier_smem") + (("packed128",) if plan.has_packed128() else ()) + (("packed_anchor",) if plan.has_packed_anchor() else ()) + (("fsm",) if plan.has_fsm() else ()):
            plan.set_path(path)
            assert np.array_equal(plan.evaluate(genomes), want), path
    plan.set_path("auto")


@pytest.mark.parametrize("case", list(_cases(DP_SUITES, "es")))
def test_decoded_partitions_match_reference(gpu, case):
    """The partition each sampled genome decodes to (reference decode_genome)
    is reproduced by both decode paths: the registry-based decode_genome and
    the device plan's replacement table."""
    g, reg, meas = build_case(case)
    res = tp.optimize(g, reg, meas, case["epsilon"])
    es = case["es"]
    plan = tp.FitnessPlan(g, reg, meas, res.placement, case["epsilon"], es["graph_backend"],
                          res.kernel_matches)
    for bits, want in zip(es["genomes"], es["decoded"]):
        a = tp.decode_genome(g, reg, res.placement, bits, es["graph_backend"])
        b = plan.decode(bits, res.placement)
        if want is None:
            assert a is None and b is None
        else:
            assert kernels_of(a) == want
            assert kernels_of(b) == want
