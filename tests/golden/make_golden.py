"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (the reference lives at /root/reference and
does not exist on the GPU box):

    python tests/golden/make_golden.py

Graphs and backend setups are drawn with this repository's own generators
(paper_2111_00655_b200.workloads and the helpers below), handed to the
reference package `tensorplace` through its JSON formats, and the
reference's outputs -- candidate matches of every node, the operator-level
DP placement and cost, graph-level costs of sampled genomes, full `evolve`
runs, and rule-generated patterns -- are written next to their inputs as
JSON.  Tests replay the inputs through the oracle and the GPU path and
compare against these outputs.
"""

from __future__ import annotations

import json
import math
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REPO)
sys.path.insert(0, REF_SRC)

import tensorplace as ref  # noqa: E402  (the reference, read-only)
from tensorplace import oracle as ref_oracle  # noqa: E402
from tensorplace.cost import profile_from_json as ref_profile_from_json  # noqa: E402
from tensorplace.cost import profile_to_json as ref_profile_to_json  # noqa: E402
from tensorplace.graph import graph_from_json as ref_graph_from_json  # noqa: E402
from tensorplace.rules import rule_to_json as ref_rule_to_json  # noqa: E402

from paper_2111_00655_b200 import workloads  # noqa: E402
from paper_2111_00655_b200.graph import graph_to_json  # noqa: E402

OPS = ("conv2d", "add", "relu", "mul", "tanh", "dense")
SHAPES = ((1, 4, 4, 4), (1, 8, 8, 8), (1, 16, 4, 4))


# -- input generators (this repository's own) ---------------------------------------------

def rand_graph_doc(rng: random.Random, n: int, ops=OPS[:4]) -> dict:
    nodes, consumed = [], set()
    for i in range(n):
        refs = []
        for _ in range(rng.choice((1, 1, 2))):
            if i and rng.random() < 0.75:
                j = rng.randrange(i)
                refs.append(j)
                consumed.add(j)
            else:
                refs.append({"input": "x"})
        nodes.append({"id": i, "op": rng.choice(ops), "attrs": {"variant": rng.randrange(3)},
                      "inputs": refs, "shape": list(rng.choice(SHAPES))})
    return {"version": "collage-graph/1", "inputs": [{"name": "x", "shape": list(SHAPES[0])}],
            "nodes": nodes, "outputs": [i for i in range(n) if i not in consumed]}


def fused_text(rng: random.Random, g) -> str | None:
    cands = [n for n in g.nodes.values() if any(isinstance(r, int) for r in n.input_ids)]
    if not cands:
        return None
    node = rng.choice(cands)
    args = [f"{g.nodes[r].op_kind}()" if isinstance(r, int) and rng.random() < 0.8 else "*"
            for r in node.input_ids]
    return f"{node.op_kind}({', '.join(args)})"


def random_setup(rng: random.Random, g, n_backends: int, ties: bool = False,
                 graph_backend: bool = False) -> dict:
    present = sorted({n.op_kind for n in g.nodes.values()})
    backends, patterns, profiles = [], [], {}
    for b in range(n_backends):
        bid = f"b{b}"
        backends.append([bid, "op_kernel_library"])
        ops = present if b == 0 else [op for op in present if rng.random() < 0.7]
        patterns += [[bid, f"{op}()", "explicit"] for op in ops]
        if b > 0 or ties:
            for _ in range(3 if ties else 2):
                t = fused_text(rng, g)
                if t is not None:
                    patterns.append([bid, t, "explicit"])
        if ties:
            table = {op: {"coeff": 0.0, "overhead": rng.choice((0.5, 1.0))} for op in present}
            disc = rng.choice((1.0, 0.5))
        else:
            table = {op: {"coeff": rng.choice((0.0, 1e-6, 2e-6)),
                          "overhead": round(rng.uniform(0.05, 1.0), 3)} for op in present}
            disc = rng.choice((1.0, 0.95, 0.9, 0.8))
        profiles[bid] = {"version": "collage-costs/1", "backend": bid, "ops": table,
                         "fusion_discount": disc}
    if graph_backend:
        backends.append(["gx", "graph_inference_library"])
        patterns += [["gx", f"{op}()", "explicit"] for op in present if rng.random() < 0.8]
        if rng.random() < 0.5:
            t = fused_text(rng, g)
            if t is not None:
                patterns.append(["gx", t, "explicit"])
        profiles["gx"] = {"version": "collage-costs/1", "backend": "gx",
                          "ops": {op: {"coeff": rng.choice((0.0, 1e-6)),
                                       "overhead": round(rng.uniform(0.05, 1.0), 3)}
                                  for op in present},
                          "region_alpha": rng.choice((0.0, 0.02, 0.05)),
                          "region_floor": rng.choice((0.7, 0.9))}
    return {"backends": backends, "patterns": patterns, "profiles": profiles}


def random_pattern_text(rng: random.Random, depth: int = 2) -> str:
    cons = ""
    if rng.random() < 0.3:
        kind = rng.randrange(3)
        if kind == 0:
            cons = "{variant=%d}" % rng.randrange(3)
        elif kind == 1:
            cons = "{variant in [0, 1]}"
        else:
            cons = "{variant in 0..%d}" % rng.randrange(1, 3)
    op = rng.choice(OPS[:4])
    if depth == 0 or rng.random() < 0.3:
        return f"{op}(){cons}"
    args = ["*" if rng.random() < 0.4 else random_pattern_text(rng, depth - 1)
            for _ in range(rng.choice((1, 2)))]
    return f"{op}({', '.join(args)}){cons}"


# -- reference drivers -------------------------------------------------------------------

def ref_registry(case: dict):
    reg = ref.PatternRegistry()
    for bid, kind in case["backends"]:
        reg.add_backend(ref.BackendDescriptor(bid, ref.BackendKind(kind)))
    for bid, text, source in case["patterns"]:
        reg.add_pattern(bid, text, ref.PatternSource(source))
    # keep exactly what was registered (duplicates are refused by the registry)
    case["patterns"] = [[bp.backend, bp.text(), bp.source.value] for bp in reg.patterns]
    measurer = ref.SimMeasurer({bid: ref_profile_from_json(doc)
                                for bid, doc in case["profiles"].items()})
    return reg, measurer


def kernels_json(placement) -> list:
    return [[a.backend_pattern.order, a.root, sorted(a.nodes)] for a in placement.assignments]


def record_candidates(g, reg) -> dict:
    out = {}
    for nid in sorted(g.nodes):
        out[str(nid)] = [[bp.order, sorted(m.nodes.node_ids),
                          [[list(pos), v] for pos, v in m.binding]]
                         for bp, m in reg.candidates_at(g, nid)]
    return out


def record_dp(g, reg, measurer, eps, max_states=50_000) -> dict:
    try:
        res = ref.optimize(g, reg, measurer, eps, max_states=max_states)
    except ref.UncoverableGraphError as exc:
        return {"error": "UncoverableGraphError", "node_ids": list(exc.node_ids),
                "op_kinds": list(exc.op_kinds)}
    except ref.SearchLimitError as exc:
        return {"error": "SearchLimitError", "message": str(exc)}
    return {"cost": res.cost_ms, "kernels": kernels_json(res.placement),
            "relaxations": res.stats.relaxations, "states_peak": res.stats.states_peak}


def record_es(g, reg, measurer, eps, dp_placement, rng: random.Random, target: str,
              n_genomes: int = 24, evolve_cfg: dict | None = None) -> dict:
    from tensorplace.evolution import eligible_slots
    k = len(eligible_slots(reg, dp_placement))
    genomes = [[0] * k, [1] * k] + [[rng.randrange(2) for _ in range(k)]
                                     for _ in range(n_genomes)]
    fits, decoded = [], []
    for bits in genomes:
        p = ref.decode_genome(g, reg, dp_placement, bits, target)
        fits.append(math.inf if p is None else ref.placement_cost_graphlevel(
            measurer, g, p, eps, reg.graph_backend_ids()))
        decoded.append(None if p is None else kernels_json(p))
    out = {"graph_backend": target, "genome_length": k, "genomes": genomes, "fitness": fits,
           "decoded": decoded}
    if evolve_cfg is not None:
        cfg = ref.ESConfig(**evolve_cfg)
        es = ref.evolve(g, reg, measurer, dp_placement, eps, cfg, graph_backend=target)
        out["evolve"] = {"config": evolve_cfg, "cost": es.cost_ms, "seed_cost": es.seed_cost_ms,
                         "history": [list(h) for h in es.history],
                         "evaluations": es.evaluations, "kernels": kernels_json(es.placement)}
        if k <= 12:
            bits, best = ref_oracle.optimal_genome(g, reg, measurer, dp_placement, eps, target)
            out["optimal_genome"] = {"bits": list(bits), "cost": best}
    return out


def make_case(name: str, graph_doc: dict, setup: dict, eps: float = 0.01) -> dict:
    return {"name": name, "graph": graph_doc, "epsilon": eps, **setup}


def build_dp_cases(seed: int, count: int, nmin: int, nmax: int, ties: bool,
                   with_es: bool = False, with_candidates: bool = True) -> list:
    rng = random.Random(seed)
    cases = []
    while len(cases) < count:
        doc = rand_graph_doc(rng, rng.randint(nmin, nmax))
        g = ref_graph_from_json(doc)
        setup = random_setup(rng, g, rng.randint(2, 3), ties=ties, graph_backend=with_es)
        eps = rng.choice((0.0, 0.25, 0.5)) if ties else 0.01
        case = make_case(f"{'tie' if ties else 'dp'}{seed}_{len(cases)}", doc, setup, eps)
        reg, measurer = ref_registry(case)
        if with_candidates:
            case["candidates"] = record_candidates(g, reg)
        case["dp"] = record_dp(g, reg, measurer, eps)
        if with_es and "kernels" in case["dp"]:
            res = ref.optimize(g, reg, measurer, eps)
            cfg = {"population_size": rng.choice((8, 16, 32)),
                   "generations": rng.choice((10, 25, 50)), "seed": rng.randrange(10_000)}
            case["es"] = record_es(g, reg, measurer, eps, res.placement, rng, "gx",
                                   evolve_cfg=cfg)
        cases.append(case)
    return cases


def matcher_cases(seed: int, count: int) -> list:
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        doc = rand_graph_doc(rng, rng.randint(2, 12))
        g = ref_graph_from_json(doc)
        texts = [random_pattern_text(rng) for _ in range(6)]
        got = {}
        for t in texts:
            got[t] = [[m.root, sorted(m.nodes.node_ids), [[list(p), v] for p, v in m.binding]]
                      for m in ref.match_all(g, ref.parse_pattern(t))]
        out.append({"name": f"match{seed}_{len(out)}", "graph": doc, "patterns": texts,
                    "matches": got})
    return out


def rule_cases(seed: int, count: int) -> list:
    from tensorplace.rules import FusionTransition, OpClass, OpValidity, PatternRule
    from tensorplace.patterns import OneOf
    rng = random.Random(seed)
    out = []
    classes = (OpClass.FUSABLE, OpClass.ELEMWISE, OpClass.INJECTIVE)
    while len(out) < count:
        doc = rand_graph_doc(rng, rng.randint(3, 12))
        g = ref_graph_from_json(doc)
        present = sorted({n.op_kind for n in g.nodes.values()})
        validity = []
        for op in present:
            if rng.random() < 0.85:
                cons = (OneOf("variant", (0, 1)),) if rng.random() < 0.25 else ()
                validity.append(OpValidity(op, cons, rng.choice(classes)))
        if not validity:
            validity.append(OpValidity(present[0], (), OpClass.FUSABLE))
        trans = tuple(FusionTransition(rng.choice(classes), rng.choice(classes),
                                       rng.choice(classes)) for _ in range(rng.randrange(1, 4)))
        rule = PatternRule("b1", tuple(validity), trans, rng.choice((2, 3, 4, 16)))
        gen = ref.generate_patterns(rule, g)
        out.append({"name": f"rule{seed}_{len(out)}", "graph": doc, "rule": ref_rule_to_json(rule),
                    "generated": [[ref.pattern_to_text(gp.pattern), gp.origin,
                                   sorted(gp.source_nodes)] for gp in gen],
                    "groups": sorted(sorted(s) for s in ref.fusion_groups(rule, g))})
    return out


def fixture_cases() -> list:
    """The reference test suite's hand-built fixtures, restated as data."""
    chain3 = {"version": "collage-graph/1",
              "inputs": [{"name": "x", "shape": [1, 16, 8, 8]}, {"name": "w", "shape": [16, 16, 3, 3]},
                         {"name": "b", "shape": [1, 16, 8, 8]}],
              "nodes": [{"id": 0, "op": "conv2d", "attrs": {"stride": 1},
                         "inputs": [{"input": "x"}, {"input": "w"}], "shape": [1, 16, 8, 8]},
                        {"id": 1, "op": "add", "attrs": {}, "inputs": [0, {"input": "b"}],
                         "shape": [1, 16, 8, 8]},
                        {"id": 2, "op": "relu", "attrs": {}, "inputs": [1], "shape": [1, 16, 8, 8]}],
              "outputs": [2]}
    unit = lambda bid, ops, o=1.0: {"version": "collage-costs/1", "backend": bid,
                                    "ops": {op: {"coeff": 0.0, "overhead": o} for op in ops}}
    two = {"backends": [["A", "op_kernel_library"], ["B", "op_kernel_library"]],
           "patterns": [["A", "conv2d()", "explicit"], ["A", "add()", "explicit"],
                        ["A", "relu()", "explicit"], ["B", "relu(add(conv2d(*, *), *))", "explicit"]],
           "profiles": {"A": unit("A", ("conv2d", "add", "relu")),
                        "B": {"version": "collage-costs/1", "backend": "B",
                              "ops": {"conv2d": {"coeff": 0.0, "overhead": 1.5},
                                      "add": {"coeff": 0.0, "overhead": 0.5},
                                      "relu": {"coeff": 0.0, "overhead": 0.5}}}}}
    tie = {"backends": [["A", "op_kernel_library"], ["B", "op_kernel_library"]],
           "patterns": [[b, f"{op}()", "explicit"] for b in "AB" for op in ("conv2d", "add", "relu")],
           "profiles": {b: unit(b, ("conv2d", "add", "relu")) for b in "AB"}}
    ops6 = ["conv2d", "add", "relu", "add", "conv2d", "conv2d"]
    chain6 = {"version": "collage-graph/1", "inputs": [{"name": "x", "shape": [1, 16, 8, 8]}],
              "nodes": [{"id": i, "op": op, "attrs": {}, "inputs": [{"input": "x"} if i == 0 else i - 1],
                         "shape": [1, 16, 8, 8]} for i, op in enumerate(ops6)], "outputs": [5]}
    offload = {"backends": [["cpu", "op_kernel_library"], ["simgraph", "graph_inference_library"]],
               "patterns": [["cpu", f"{op}()", "explicit"] for op in ("conv2d", "add", "relu")]
               + [["simgraph", f"{op}()", "explicit"] for op in ("add", "relu")],
               "profiles": {"cpu": unit("cpu", ("conv2d", "add", "relu")),
                            "simgraph": {**unit("simgraph", ("add", "relu"), 1.02),
                                         "region_alpha": 0.05, "region_floor": 0.7}}}
    cases = [make_case("fixture_fused_chain", chain3, two), make_case("fixture_tie", chain3, tie),
             make_case("fixture_offload_chain", chain6, offload)]
    for c in cases:
        reg, meas = ref_registry(c)
        g = ref_graph_from_json(c["graph"])
        c["candidates"] = record_candidates(g, reg)
        c["dp"] = record_dp(g, reg, meas, c["epsilon"])
    c = cases[2]
    reg, meas = ref_registry(c)
    g = ref_graph_from_json(c["graph"])
    res = ref.optimize(g, reg, meas, 0.01)
    c["es"] = record_es(g, reg, meas, 0.01, res.placement, random.Random(7), "simgraph",
                        evolve_cfg={"population_size": 16, "generations": 40, "seed": 0})
    return cases


def model_case(name: str, g_mine, backend_set, eps: float = 0.01, es_cfg=None,
               max_states: int = 200_000) -> dict:
    doc = graph_to_json(g_mine)
    reg_mine = backend_set.registry
    setup = {"backends": [[b.id, b.kind.value] for b in reg_mine.backends.values()],
             "patterns": [[bp.backend, bp.text(), bp.source.value] for bp in reg_mine.patterns],
             "profiles": {bid: ref_profile_to_json(ref_profile_from_json(
                 _mine_profile_json(p))) for bid, p in backend_set.measurer.profiles.items()}}
    case = make_case(name, doc, setup, eps)
    g = ref_graph_from_json(doc)
    reg, meas = ref_registry(case)
    t0 = time.time()
    case["dp"] = record_dp(g, reg, meas, eps, max_states=max_states)
    case["dp"]["reference_seconds"] = time.time() - t0
    if es_cfg is not None and "kernels" in case["dp"]:
        res = ref.optimize(g, reg, meas, eps, max_states=max_states)
        case["es"] = record_es(g, reg, meas, eps, res.placement, random.Random(11),
                               backend_set.graph_backend, n_genomes=16, evolve_cfg=es_cfg)
    return case


def _mine_profile_json(p) -> dict:
    from paper_2111_00655_b200.cost import profile_to_json
    return profile_to_json(p)


def main() -> None:
    out_dir = HERE
    t0 = time.time()
    suites = {
        "fixtures": fixture_cases(),
        "dp_random": build_dp_cases(101, 120, 3, 12, ties=False),
        "dp_ties": build_dp_cases(202, 100, 3, 14, ties=True),
        "dp_large": build_dp_cases(303, 12, 20, 40, ties=False, with_candidates=False),
        "es_random": build_dp_cases(404, 50, 3, 10, ties=False, with_es=True,
                                    with_candidates=False),
        "matcher": matcher_cases(505, 60),
        "rules": rule_cases(606, 60),
    }
    for name, cases in suites.items():
        with open(os.path.join(out_dir, f"{name}.json"), "w") as fh:
            json.dump(cases, fh, separators=(",", ":"))
        print(f"{name}: {len(cases)} cases ({time.time() - t0:.1f}s)", flush=True)
    models = []
    for model, fn in (("resnet50", workloads.resnet50), ("bert_base", workloads.bert_base),
                      ("nasrnn", lambda: workloads.nasrnn(steps=1))):
        g = fn()
        bs = workloads.paper_backends(g, verify=False)
        # the rule expansion must agree with the reference generator
        rg = ref_graph_from_json(graph_to_json(g))
        from tensorplace.rules import rule_from_json as ref_rule_from_json
        from paper_2111_00655_b200.rules import rule_to_json as my_rule_to_json
        ref_gen = ref.generate_patterns(ref_rule_from_json(my_rule_to_json(bs.rules["tvm"])), rg)
        from paper_2111_00655_b200.rules import generate_patterns as my_gen
        mine = my_gen(bs.rules["tvm"], g, verify=False)
        assert [ref.pattern_to_text(x.pattern) for x in ref_gen] == \
            [__import__("paper_2111_00655_b200").pattern_to_text(x.pattern) for x in mine], model
        models.append(model_case(model, g, bs, es_cfg={"population_size": 16, "generations": 10,
                                                       "seed": 1}))
        print(f"model {model}: dp {models[-1]['dp'].get('cost', models[-1]['dp'])} "
              f"({time.time() - t0:.1f}s)", flush=True)
    with open(os.path.join(out_dir, "models.json"), "w") as fh:
        json.dump(models, fh, separators=(",", ":"))


if __name__ == "__main__":
    main()
