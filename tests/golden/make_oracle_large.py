"""Fixtures for graphs beyond the reference DP's state cap, solved by the CPU
oracle's covered-set DP (oracle/oracle.c, the reference's Algorithm 1
restated and pinned to the reference on every golden case) with a 30 M-state
cap.  Run in the build container:

    python tests/golden/make_oracle_large.py

Writes tests/golden/oracle_large.json: the case (graph, backends, patterns,
profiles) and the oracle's optimum (cost, kernels).  NasRNN with one step
(47 nodes) needs ~10 s here; the reference Python DP gives up on it at
200 000 live states.
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

from oracle import OracleCase  # noqa: E402  (checker)
from paper_2111_00655_b200 import workloads  # noqa: E402
from paper_2111_00655_b200.cost import profile_to_json  # noqa: E402
from paper_2111_00655_b200.graph import graph_to_json  # noqa: E402


def case_of(name, g, bs, eps=0.01):
    return json.loads(json.dumps({
        "name": name, "graph": graph_to_json(g), "epsilon": eps,
        "backends": [[b.id, b.kind.value] for b in bs.registry.backends.values()],
        "patterns": [[bp.backend, bp.text(), bp.source.value] for bp in bs.registry.patterns],
        "profiles": {b: profile_to_json(p) for b, p in bs.measurer.profiles.items()}}))


def main():
    out = []
    g = workloads.nasrnn(steps=1)
    bs = workloads.paper_backends(g, verify=False)
    case = case_of("nasrnn_1step", g, bs)
    oc = OracleCase(case)
    oc.price()
    t0 = time.time()
    status, cost, kernels = oc.dp(max_states=30_000_000)
    assert status == "ok", status
    case["oracle_dp"] = {"status": status, "cost": cost, "kernels": kernels,
                         "max_states": 30_000_000, "seconds": time.time() - t0}
    out.append(case)
    with open(os.path.join(HERE, "oracle_large.json"), "w") as fh:
        json.dump(out, fh)
    print("wrote", len(out), "cases")


if __name__ == "__main__":
    main()
