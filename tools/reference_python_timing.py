"""Time the REFERENCE Python package (tensorplace, /root/reference) on the
bench configs -- build container only (the reference does not travel to the
GPU box).  Writes profiles/r01_reference_python.json:

* DP (`tensorplace.optimize`) wall time per config (or its failure);
* graph-level fitness of random genomes (decode_genome +
  placement_cost_graphlevel, what each ES evaluation does), one core;
* the reference's full search with its default ES config (DP + evolve,
  population 32, 200 generations) where the DP finishes.
"""
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(REPO, "tests", "golden"))
import make_golden as mg  # noqa: E402  (reference import + JSON bridges)
from make_golden import ref  # noqa: E402
from paper_2111_00655_b200 import workloads  # noqa: E402

out = {}
for name in sys.argv[1:] or ["resnet50", "bert_base", "nasnet_a", "nasrnn"]:
    g_mine = workloads.CONFIGS[name]()
    bs = workloads.paper_backends(g_mine, verify=False)
    case = mg.model_case(name, g_mine, bs)
    g = mg.ref_graph_from_json(case["graph"])
    reg, meas = mg.ref_registry(case)
    row = {"dp": {k: v for k, v in case["dp"].items() if k != "kernels"}}
    if "kernels" in case["dp"]:
        res = ref.optimize(g, reg, meas, 0.01, max_states=200_000)
        from tensorplace.evolution import eligible_slots
        k = len(eligible_slots(reg, res.placement))
        rng = random.Random(0)
        genomes = [[rng.randrange(2) for _ in range(k)] for _ in range(200)]
        t0 = time.perf_counter()
        for bits in genomes:
            p = ref.decode_genome(g, reg, res.placement, bits, bs.graph_backend)
            if p is not None:
                ref.placement_cost_graphlevel(meas, g, p, 0.01, reg.graph_backend_ids())
        dt = time.perf_counter() - t0
        row["fitness_genomes_per_s_1core"] = len(genomes) / dt
        t0 = time.perf_counter()
        res = ref.optimize(g, reg, meas, 0.01, max_states=200_000)
        es = ref.evolve(g, reg, meas, res.placement, 0.01, ref.ESConfig(),
                        graph_backend=bs.graph_backend)
        row["search_default_es_s"] = time.perf_counter() - t0
        row["search_default_es"] = {"population": 32, "generations": 200,
                                    "evaluations": es.evaluations, "cost_ms": es.cost_ms,
                                    "dp_cost_ms": res.cost_ms}
    out[name] = row
    print(name, json.dumps(row), flush=True)
json.dump(out, open(os.path.join(REPO, "profiles", "r01_reference_python.json"), "w"), indent=1)
