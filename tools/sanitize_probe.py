"""Small end-to-end exercise of every device path, for compute-sanitizer:
matcher, pricing, DP (narrow + wide launches), every fitness kernel, breed,
fused generation, argmin."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads
from paper_2111_00655_b200.es_device import DeviceEvolution

# CB_FSM_ENTRY_BYTES=16 / 32 in the environment selects the FSM walk's
# wider transition layouts; "narrow" (a long DAG with few slots) runs the
# FSM walk with genome words loaded on demand (W = 0)
for name, g, bs in (
        ("bert", workloads.bert_base(layers=1), None),
        ("rand", workloads.random_dag(400, seed=2, ops=workloads.RANDOM_OPS, window=48), None),
        ("narrow", workloads.random_dag(700, seed=9, ops=workloads.RANDOM_OPS, window=6), None),
        ("nasnet", workloads.nasnet_a(), None)):  # the mixed 8 / 16-byte FSM layout
    bs = workloads.paper_backends(g, verify=False) if name in ("bert", "nasnet") else \
        workloads.random_backends(g, n_backends=6, n_graph=1, seed=2 if name == "rand" else 9)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
    plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                          res.kernel_matches)
    rng = np.random.default_rng(0)
    genomes = (rng.random((97, plan.k)) < 0.5).astype(np.uint8)
    want = None
    paths = ["auto", "unionfind", "wide"] + (["anchor"] if plan.info.window_shift >= 0 else [])
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
        got = plan.evaluate(genomes)
        if want is None:
            want = got
        assert np.array_equal(got, want), (name, path)
    plan.set_path("auto")
    if plan.info.window_shift >= 0:
        plan.set_path("anchor")
        plan.set_pool(1)
        assert np.array_equal(plan.evaluate(genomes), want)
        plan.set_pool(16)
        plan.set_path("auto")
    for fused in (False, True):
        es = DeviceEvolution(plan, 300, seed=1, fused=fused)
        es.initialize()
        for _ in range(3):
            es.step()
        es.best()
    print(name, plan.info.frontier_slots, "words", plan.words, "fsm entry bytes", plan.info.fsm_entry_bytes,
          paths, "ok", flush=True)
