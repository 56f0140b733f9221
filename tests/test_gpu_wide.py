"""Wide frontier programs (17..128 slots: random DAGs with long-range
edges, like the 100k-op config) evaluated by the sparse warp-per-genome
kernel, bit-exact against the CPU oracle (oracle/oracle.c, the reference's
graph-level pricing restated) and against the union-find kernels."""

import json

import numpy as np
import pytest

import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads
from paper_2111_00655_b200.cost import profile_to_json
from paper_2111_00655_b200.graph import graph_to_json
from oracle import OracleCase

pytestmark = pytest.mark.gpu


def _case(g, bs, eps):
    return json.loads(json.dumps({
        "graph": graph_to_json(g),
        "backends": [[b.id, b.kind.value] for b in bs.registry.backends.values()],
        "patterns": [[bp.backend, bp.text(), bp.source.value] for bp in bs.registry.patterns],
        "profiles": {b: profile_to_json(p) for b, p in bs.measurer.profiles.items()},
        "epsilon": eps}))


def _genomes(plan, rng, rows_per_density=300):
    feasible = np.array([k != 0 for k in plan.rep_kind], dtype=np.uint8)
    rows = []
    for d in (0.02, 0.1, 0.3, 0.5, 0.8, 1.0):
        x = (rng.random((rows_per_density, plan.k)) < d).astype(np.uint8)
        x[: rows_per_density // 2] &= feasible  # half guaranteed feasible
        rows.append(x)
    rows.append(np.zeros((1, plan.k), np.uint8))
    rows.append(feasible[None, :])
    return np.concatenate(rows)


@pytest.mark.parametrize("seed,n,window", [(0, 2000, 64), (1, 3000, 64), (2, 1500, 128),
                                           (3, 800, 24)])
def test_wide_plan_matches_oracle(gpu, seed, n, window, monkeypatch):
    g = workloads.random_dag(n, seed=seed, ops=workloads.RANDOM_OPS, window=window)
    bs = workloads.random_backends(g, n_backends=8, n_graph=1, seed=seed)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
    plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                          res.kernel_matches)
    ug = plan.unit_graph()
    assert plan.info.frontier_slots == ug["frontier_needed"]
    genomes = _genomes(plan, np.random.default_rng(seed))
    oc = OracleCase(_case(g, bs, 0.01))
    oc.price()
    kernels = [[a.backend_pattern.order, a.root, sorted(a.nodes)]
               for a in res.placement.assignments]
    want = oc.fitness(kernels, bs.graph_backend, genomes, threads=8)
    got = plan.evaluate(genomes)  # auto: wide kernel for > 16 slots
    assert np.array_equal(got, want)
    for path in ("wide", "anchor"):
        plan.set_path(path)
        assert np.array_equal(plan.evaluate(genomes), want), path
    # the anchor walk's launch forms: 64- / 128-thread blocks, merges with
    # selects or branches (chosen by population size; forced here)
    for block in ("64", "128"):
        for merge in ("0", "1"):
            monkeypatch.setenv("CB_ANCHOR_BLOCK", block)
            monkeypatch.setenv("CB_ANCHOR_MERGE", merge)
            assert np.array_equal(plan.evaluate(genomes), want), (block, merge)
    monkeypatch.delenv("CB_ANCHOR_BLOCK")
    monkeypatch.delenv("CB_ANCHOR_MERGE")
    # tiny shared pools: merged sums spill to the thread's local memory
    for entries in (1, 2, 5):
        plan.set_pool(entries)
        assert np.array_equal(plan.evaluate(genomes), want), entries
    plan.set_pool(16)
    plan.set_path("unionfind")
    assert np.array_equal(plan.evaluate(genomes), want)
    plan.set_path("auto")


@pytest.mark.parametrize("name", ["resnet50", "bert_base", "nasnet_a", "nasrnn"])
def test_wide_kernel_agrees_on_models(gpu, name):
    g = workloads.CONFIGS[name]()
    bs = workloads.paper_backends(g)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
    plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                          res.kernel_matches)
    genomes = _genomes(plan, np.random.default_rng(5), 2000)
    plan.set_path("auto")
    want = plan.evaluate(genomes)
    for path in ("wide", "anchor", "frontier") + (("packed128",) if plan.has_packed128() else ()) + (("packed_anchor",) if plan.has_packed_anchor() else ()) + (("fsm",) if plan.has_fsm() else ()):
        plan.set_path(path)
        assert np.array_equal(plan.evaluate(genomes), want), path
    plan.set_path("auto")


def test_plan_outside_the_128_bit_window_uses_192_bit_kernels(gpu):
    """Costs spanning ~160 bits (1e-18 .. 1e12 ms) leave no 128-bit window:
    the automatic path falls back to the 192-bit walks, still bit-exact."""
    from paper_2111_00655_b200.cost import OpCost, SimMeasurer, SimProfile
    g = workloads.random_dag(300, seed=4, ops=workloads.RANDOM_OPS, window=16)
    bs = workloads.random_backends(g, n_backends=4, n_graph=1, seed=4)
    profiles = {}
    for bid, p in bs.measurer.profiles.items():
        scale = 1e12 if bid == bs.graph_backend else 1e-18
        profiles[bid] = SimProfile(bid, {op: OpCost(0.0, oc.overhead * scale)
                                         for op, oc in p.op_costs.items()},
                                   fusion_discount=p.fusion_discount, region_alpha=p.region_alpha,
                                   region_floor=p.region_floor)
    meas = SimMeasurer(profiles)
    res = tp.optimize(g, bs.registry, meas, 0.01, rounding="exact")
    plan = tp.FitnessPlan(g, bs.registry, meas, res.placement, 0.01, bs.graph_backend,
                          res.kernel_matches)
    assert plan.k > 0
    assert plan.info.window_shift == -1 and not plan.has_packed128()
    genomes = _genomes(plan, np.random.default_rng(9), 200)
    class _B:  # the oracle reads profiles from the backend set
        registry, measurer = bs.registry, meas
    oc = OracleCase(_case(g, _B, 0.01))
    oc.price()
    kernels = [[a.backend_pattern.order, a.root, sorted(a.nodes)] for a in res.placement.assignments]
    want = oc.fitness(kernels, bs.graph_backend, genomes)
    assert np.array_equal(plan.evaluate(genomes), want)
    assert plan.kernel_name() in ("fitness_frontier2_kernel", "fitness_wide_kernel",
                                  "fitness_frontier_kernel")
    for path in ("unionfind", "wide"):
        plan.set_path(path)
        assert np.array_equal(plan.evaluate(genomes), want), path
    plan.set_path("auto")


def _scaled(bs, scale_of):
    from paper_2111_00655_b200.cost import OpCost, SimMeasurer, SimProfile
    return SimMeasurer({bid: SimProfile(bid, {op: OpCost(oc.coeff, oc.overhead * scale_of(bid))
                                              for op, oc in p.op_costs.items()},
                                        fusion_discount=p.fusion_discount,
                                        region_alpha=p.region_alpha, region_floor=p.region_floor)
                        for bid, p in bs.measurer.profiles.items()})


@pytest.mark.parametrize("n_rows", [1, 31, 33, 1000])
def test_edge_plans_every_path(gpu, n_rows):
    """Degenerate plans through every kernel path, against the oracle:
    no genome bits (everything on the graph backend), every kernel offloadable
    with a cheap graph backend (long regions), and odd population sizes."""
    g = workloads.random_dag(200, seed=6, ops=workloads.RANDOM_OPS, window=12)
    bs = workloads.random_backends(g, n_backends=4, n_graph=1, seed=6)
    for name, scale in (("all-graph", lambda b: 1e-3 if b == bs.graph_backend else 1.0),
                        ("cheap-graph", lambda b: 0.5 if b == bs.graph_backend else 1.0),
                        ("no-graph", lambda b: 1e3 if b == bs.graph_backend else 1.0)):
        meas = _scaled(bs, scale)
        res = tp.optimize(g, bs.registry, meas, 0.01, rounding="exact")
        plan = tp.FitnessPlan(g, bs.registry, meas, res.placement, 0.01, bs.graph_backend,
                              res.kernel_matches)
        assert (plan.k == 0) == (name == "all-graph"), (name, plan.k)
        rng = np.random.default_rng(n_rows)
        genomes = (rng.random((n_rows, plan.k)) < 0.5).astype(np.uint8)

        class _B:
            registry, measurer = bs.registry, meas
        oc = OracleCase(_case(g, _B, 0.01))
        oc.price()
        kernels = [[a.backend_pattern.order, a.root, sorted(a.nodes)]
                   for a in res.placement.assignments]
        want = oc.fitness(kernels, bs.graph_backend, genomes)
        paths = ["auto", "unionfind"]
        if plan.info.frontier_slots:
            paths += ["wide", "anchor"] if plan.info.window_shift >= 0 else ["wide"]
        if 0 < plan.info.frontier_slots <= 32:
            paths += ["frontier", "frontier_smem"]
        if plan.has_packed128():
            paths.append("packed128")
        if plan.has_packed_anchor():
            paths.append("packed_anchor")
        if plan.has_fsm():
            paths.append("fsm")
        for path in paths:
            plan.set_path(path)
            assert np.array_equal(plan.evaluate(genomes), want), (name, path)
        plan.set_path("auto")


@pytest.mark.parametrize("name", ["bert_base", "nasrnn", "nasnet_a"])
def test_fsm_entry_layouts_agree(gpu, name, monkeypatch):
    """The 8-byte and 16-byte transition layouts (shared delta table) and the
    32-byte one (chosen by CB_FSM_ENTRY_BYTES at plan build) give identical
    fitness; NasNet-A (up to 5 merges per transition in 16 of its 620 steps)
    gets the mixed layout: 8-byte transitions except in those steps."""
    g = workloads.CONFIGS[name]()
    bs = workloads.paper_backends(g)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
    args = (g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend, res.kernel_matches)
    plans = {}
    for nbytes in (8, 16, 32):
        monkeypatch.setenv("CB_FSM_ENTRY_BYTES", str(nbytes))
        plans[nbytes] = tp.FitnessPlan(*args)
    monkeypatch.delenv("CB_FSM_ENTRY_BYTES")
    default = tp.FitnessPlan(*args)
    monkeypatch.setenv("CB_FSM_D64", "0")
    plans["d128"] = tp.FitnessPlan(*args)  # the 16-byte shared delta table
    monkeypatch.delenv("CB_FSM_D64")
    assert plans["d128"].kernel_name().endswith(", 3>" if name == "nasnet_a" else ", 1>")
    assert all(p.has_fsm() for p in plans.values())
    want_small = 8
    assert default.info.fsm_entry_bytes == want_small
    # layout 3 (mixed) for NasNet-A, 1 (8 bytes) otherwise; + 4: 8-byte deltas
    assert default.kernel_name().endswith(", 7>" if name == "nasnet_a" else ", 5>")
    assert plans[8].info.fsm_entry_bytes == want_small
    assert plans[16].info.fsm_entry_bytes == 16 and plans[32].info.fsm_entry_bytes == 32
    assert len({p.info.fsm_transitions for p in plans.values()}) == 1
    genomes = _genomes(plans[8], np.random.default_rng(11), 1000 if name == "nasnet_a" else 4000)
    plans[32].set_path("unionfind")
    want = plans[32].evaluate(genomes)
    for nbytes, plan in plans.items():
        plan.set_path("fsm")
        assert np.array_equal(plan.evaluate(genomes), want), nbytes
    assert default.kernel_name().startswith("fitness_fsm_kernel")  # automatic choice


@pytest.mark.parametrize("seed,n,window", [(7, 1200, 4), (8, 2500, 3), (9, 700, 6), (10, 400, 8)])
def test_fsm_long_narrow_programs_match_oracle(gpu, seed, n, window):
    """Long, narrow random DAGs: many genome words (the FSM kernel's W = 0
    path, words loaded on demand) with few frontier slots, every transition
    layout, against the oracle."""
    g = workloads.random_dag(n, seed=seed, ops=workloads.RANDOM_OPS, window=window)
    bs = workloads.random_backends(g, n_backends=6, n_graph=1, seed=seed)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
    plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                          res.kernel_matches)
    if not plan.has_fsm():
        pytest.skip(f"no FSM program ({plan.info.frontier_slots} slots)")
    genomes = _genomes(plan, np.random.default_rng(seed), 200)
    oc = OracleCase(_case(g, bs, 0.01))
    oc.price()
    kernels = [[a.backend_pattern.order, a.root, sorted(a.nodes)]
               for a in res.placement.assignments]
    want = oc.fitness(kernels, bs.graph_backend, genomes, threads=8)
    plan.set_path("fsm")
    assert np.array_equal(plan.evaluate(genomes), want), (plan.words, plan.info.fsm_entry_bytes)
    plan.set_path("auto")
    assert np.array_equal(plan.evaluate(genomes), want)


@pytest.mark.parametrize("n_nodes,window", [(12, 4), (40, 8), (300, 24)])
def test_anchor_walk_small_programs_and_batches(gpu, n_nodes, window, monkeypatch):
    """Programs shorter than one staged record chunk (32 steps), batches of
    1..33 genomes (partial warps and blocks), every launch form."""
    g = workloads.random_dag(n_nodes, seed=n_nodes, ops=workloads.RANDOM_OPS, window=window)
    bs = workloads.random_backends(g, n_backends=5, n_graph=1, seed=n_nodes)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
    plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                          res.kernel_matches)
    if plan.info.window_shift < 0 or plan.info.frontier_slots == 0:
        pytest.skip("no anchor program for this plan")
    oc = OracleCase(_case(g, bs, 0.01))
    oc.price()
    kernels = [[a.backend_pattern.order, a.root, sorted(a.nodes)]
               for a in res.placement.assignments]
    rng = np.random.default_rng(n_nodes)
    feasible = np.array([k != 0 for k in plan.rep_kind], dtype=np.uint8)
    plan.set_path("anchor")
    for n in (1, 2, 31, 33):
        genomes = (rng.random((n, plan.k)) < 0.5).astype(np.uint8) & feasible
        want = oc.fitness(kernels, bs.graph_backend, genomes, threads=4)
        for block in ("64", "128"):
            monkeypatch.setenv("CB_ANCHOR_BLOCK", block)
            assert np.array_equal(plan.evaluate(genomes), want), (n, block)
    plan.set_path("auto")
