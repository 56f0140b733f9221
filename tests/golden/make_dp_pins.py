"""DP placements of the five BASELINE.json configs, pinned by the oracle's
independent exact solver (oracle/oracle.c or_dp_subtree).

The reference Python DP (tensorplace/dp.py:71-179) gives up on NasNet-A,
the 10-step NasRNN and the 100k-node random DAG (SearchLimitError), and the
oracle's covered-set restatement of it cannot finish them either.
or_dp_subtree computes the same optimum by a different method (post-
dominator subtree recursion with the reference's literal post-dominator
sets, Kulisch sums and materialised canonical keys); it is checked equal
to the reference on every golden DP case and to the covered-set oracle on
the cases beyond the reference's cap (tests/test_oracle_golden.py).  A pin
also records the smallest positive decision regret: when it is at least
4 ulp of the cost, the reference's rounded comparisons provably choose the
same partition (oracle.window_safe).

Run in the build container:

    python tests/golden/make_dp_pins.py

Writes tests/golden/cases/<config>.json.gz (the case: graph, backends,
patterns, profiles -- also the input of bench.py's reference arm, which
must not load the product library) and tests/golden/dp_pins.json.
"""
import gzip
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

from oracle import OracleCase, window_safe  # noqa: E402  (checker)
from paper_2111_00655_b200 import workloads  # noqa: E402
from paper_2111_00655_b200.cost import profile_to_json  # noqa: E402
from paper_2111_00655_b200.graph import graph_to_json  # noqa: E402

CONFIGS = ["resnet50", "bert_base", "nasnet_a", "nasrnn", "random100k"]


def digest(obj) -> str:
    return hashlib.sha256(json.dumps(obj, separators=(",", ":")).encode()).hexdigest()


def case_of(name: str) -> dict:
    g = workloads.CONFIGS[name]()
    bs = workloads.random_backends(g, n_backends=8, n_graph=1, seed=0) if name == "random100k" \
        else workloads.paper_backends(g, verify=False)
    return json.loads(json.dumps({
        "name": name, "graph": graph_to_json(g), "epsilon": 0.01,
        "backends": [[b.id, b.kind.value] for b in bs.registry.backends.values()],
        "patterns": [[bp.backend, bp.text(), bp.source.value] for bp in bs.registry.patterns],
        "profiles": {b: profile_to_json(p) for b, p in bs.measurer.profiles.items()},
        "graph_backend": bs.graph_backend}))


def main():
    os.makedirs(os.path.join(HERE, "cases"), exist_ok=True)
    pins = {}
    for name in CONFIGS:
        t0 = time.time()
        case = case_of(name)
        with gzip.open(os.path.join(HERE, "cases", f"{name}.json.gz"), "wt") as fh:
            json.dump(case, fh, separators=(",", ":"))
        oc = OracleCase(case)
        oc.price()
        status, cost, kernels, regret = oc.dp_subtree()
        assert status == "ok", (name, status)
        pin = {"case_sha256": digest(case), "nodes": len(case["graph"]["nodes"]),
               "candidates": int(oc._mt["n"]), "cost": cost, "n_kernels": len(kernels),
               "kernels_sha256": digest(kernels), "min_regret": regret,
               "window_safe": window_safe(cost, regret), "exact_ties": oc.subtree_ties,
               "solver": "oracle/oracle.c or_dp_subtree", "seconds": round(time.time() - t0, 2)}
        if len(kernels) <= 1000:
            pin["kernels"] = kernels
        pins[name] = pin
        print(name, {k: v for k, v in pin.items() if k != "kernels"}, flush=True)
    with open(os.path.join(HERE, "dp_pins.json"), "w") as fh:
        json.dump(pins, fh, indent=1)


if __name__ == "__main__":
    main()
