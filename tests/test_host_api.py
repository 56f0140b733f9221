"""Host-side API (no GPU): DSL, graph validation, file formats, rule
expansion, registry semantics, genome packing."""

import json
import random

import numpy as np
import pytest

import paper_2111_00655_b200 as tp
from conftest import golden
from paper_2111_00655_b200.evolution import pack_genomes
from paper_2111_00655_b200.rules import rule_from_json, rule_to_json


def test_pattern_round_trip_and_errors():
    texts = ['conv2d(*, *){data_layout="NCHW"}', "relu(add(conv2d(*, *), *))",
             "dense(*){units in 1..4096}", 'add(*, *){dtype in ["f16", "f32"], k=2.5}', "relu()"]
    for t in texts:
        p = tp.parse_pattern(t)
        assert tp.parse_pattern(tp.pattern_to_text(p)) == p
    for bad, col in (("conv2d(*,", 10), ("*", 1), ("relu(*) x", 9), ("a(){k in 3..1}", 13)):
        with pytest.raises(tp.PatternSyntaxError) as info:
            tp.parse_pattern(bad)
        assert info.value.line == 1 and info.value.column == col, bad


def test_graph_validation_errors():
    I = tp.InputRef("x")
    with pytest.raises(tp.GraphValidationError) as info:
        tp.ComputationGraph([tp.GraphInput("x", (4,))],
                            [tp.OperatorNode(0, "relu", {}, (99,), (4,))], [0])
    assert "99" in str(info.value)
    with pytest.raises(tp.GraphValidationError) as info:
        tp.ComputationGraph([tp.GraphInput("x", (4,))],
                            [tp.OperatorNode(0, "add", {}, (I, 1), (4,)),
                             tp.OperatorNode(1, "relu", {}, (0,), (4,))], [1])
    assert info.value.node_id == 0
    with pytest.raises(tp.GraphValidationError):
        tp.ComputationGraph([tp.GraphInput("x", (4,))],
                            [tp.OperatorNode(0, "relu", {}, (I,), (4,)),
                             tp.OperatorNode(1, "relu", {}, (I,), (4,))], [1])
    with pytest.raises(tp.GraphValidationError):
        tp.ComputationGraph([tp.GraphInput("x", (0,))], [], [])
    assert tp.ComputationGraph([], [], []).topo_order() == ()


def test_graph_json_round_trip(tmp_path):
    from paper_2111_00655_b200 import workloads
    for g in (workloads.resnet50(), workloads.random_dag(40, seed=3)):
        p1, p2 = tmp_path / "a.json", tmp_path / "b.json"
        tp.save_graph(g, str(p1))
        g1 = tp.load_graph(str(p1))
        tp.save_graph(g1, str(p2))
        assert tp.load_graph(str(p2)) == g1 == g
    with pytest.raises(tp.GraphFormatError):
        tp.graph_from_json({"version": "nope", "inputs": [], "nodes": [], "outputs": []})


def test_rule_expansion_matches_reference_on_host():
    """Host-side growth (without the device self-check) equals the
    reference generator on every golden rule case."""
    for case in golden("rules"):
        g = tp.graph_from_json(case["graph"])
        rule = rule_from_json(case["rule"])
        gen = tp.generate_patterns(rule, g, verify=False)
        assert [[tp.pattern_to_text(x.pattern), x.origin, sorted(x.source_nodes)]
                for x in gen] == case["generated"], case["name"]
        assert sorted(sorted(s) for s in tp.fusion_groups(rule, g)) == case["groups"]
        assert rule_from_json(json.loads(json.dumps(rule_to_json(rule)))) == rule


def test_registry_semantics():
    reg = tp.PatternRegistry()
    reg.add_backend(tp.BackendDescriptor("a", tp.BackendKind.OP_KERNEL_LIBRARY))
    with pytest.raises(tp.RegistryError):
        reg.add_backend(tp.BackendDescriptor("a", tp.BackendKind.OP_KERNEL_LIBRARY))
    with pytest.raises(tp.RegistryError):
        reg.add_pattern("zzz", "relu()")
    assert reg.add_pattern("a", "relu()") is True
    assert reg.add_pattern("a", "relu()") is False
    assert [bp.order for bp in reg.patterns] == [0]
    clone = tp.PatternRegistry.from_json(reg.to_json())
    assert [bp.text() for bp in clone.patterns] == ["relu()"]


def test_file_formats_round_trip(tmp_path):
    prof = tp.SimProfile("cpu", {"relu": tp.OpCost(1e-6, 0.01)}, fusion_discount=0.9,
                         region_alpha=0.02, region_floor=0.8)
    tp.save_profile(prof, str(tmp_path / "p.json"))
    assert tp.load_profile(str(tmp_path / "p.json")) == prof
    (tmp_path / "c.jsonl").write_text('{"key": "a", "cost_ms": 1.5}\nnot json\n'
                                      '{"key": "b", "cost_ms": 2.0}\n')
    cache = tp.cache_load(str(tmp_path / "c.jsonl"))
    assert len(cache) == 2 and len(cache.load_warnings) == 1
    tp.cache_save(cache, str(tmp_path / "d.jsonl"))
    assert dict(tp.cache_load(str(tmp_path / "d.jsonl")).items()) == dict(cache.items())
    with pytest.raises(tp.CacheFormatError):
        tp.cache_load(str(tmp_path / "missing.jsonl"))
    pats = [tp.parse_pattern(t) for t in ("relu(add(*, *))", "dense()")]
    tp.save_pattern_file(pats, str(tmp_path / "k.pat"), comments=["x", "y"])
    assert tp.load_pattern_file(str(tmp_path / "k.pat")) == pats


def test_kernel_cost_and_totals_follow_fsum():
    g = tp.graph_from_json(golden("fixtures")[0]["graph"])
    prof = tp.SimProfile("B", {"conv2d": tp.OpCost(0.0, 1.5), "add": tp.OpCost(0.0, 0.5),
                               "relu": tp.OpCost(1e-6, 0.5)}, fusion_discount=0.9)
    sub = tp.Subgraph(g, frozenset(g.nodes))
    vol = 16 * 8 * 8
    assert prof.kernel_cost(sub) == (1.5 + 0.5 + (1e-6 * vol + 0.5)) * 0.9 ** 2
    assert tp.total_cost([1.0, 2.0], 0.01) == 3.02


def test_genome_packing_layout():
    rng = np.random.default_rng(0)
    for k in (1, 63, 64, 65, 185):
        bits = rng.integers(0, 2, size=(5, k), dtype=np.uint8)
        words = (k + 63) // 64
        packed = pack_genomes(bits, k, words)
        for r in range(5):
            for i in range(k):
                assert (int(packed[r, i // 64]) >> (i % 64)) & 1 == bits[r, i]


def test_es_config_validation():
    for kw in ({"population_size": 0}, {"generations": -1}, {"mutation_rate": 1.5},
               {"tournament_size": 0}, {"time_budget_s": 0.0}):
        with pytest.raises(ValueError):
            tp.ESConfig(**kw)
