"""Near-tie cases for the rounding window, solved by the REFERENCE.

The reference compares covered-set states by rounded costs
(tensorplace/dp.py:128-147); the device compares exact sums.  These cases
put an alternative partition within one ulp of the optimum, so the two
can disagree.  `optimize` must refuse to certify them (RoundingWindowError)
instead of silently returning a placement the reference would not.

    python tests/golden/make_rounding_golden.py   (build container only)
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import ref, ref_graph_from_json, ref_registry, record_dp  # noqa: E402
from tensorplace.cost import COSTS_FORMAT_VERSION  # noqa: E402


def profile(bid, ops, discount=1.0):
    return {"version": COSTS_FORMAT_VERSION, "backend": bid, "fusion_discount": discount,
            "region_alpha": 0.05, "region_floor": 0.7,
            "ops": {op: {"coeff": 0.0, "overhead": o} for op, o in ops.items()}}


def chain(ops):
    nodes = []
    for i, op in enumerate(ops):
        nodes.append({"id": i, "op": op, "attrs": {}, "inputs": [i - 1] if i else [{"input": "x"}],
                      "shape": [1, 4]})
    return {"version": "collage-graph/1", "inputs": [{"name": "x", "shape": [1, 4]}],
            "nodes": nodes, "outputs": [len(ops) - 1]}


def main():
    cases = []
    # 0.1 + 0.2 as two kernels (exact 0.30000000000000001665) against one
    # fused kernel priced round(0.1 + 0.2) = 0.30000000000000004441: with
    # epsilon 0 both round to the same total and the reference takes the
    # smaller key, which is the fused pattern when it is registered first.
    for name, fused_first, eps in (("fused_key_wins", True, 0.0), ("singles_key_wins", False, 0.0),
                                   ("epsilon_separates", True, 0.01)):
        pats = [["b0", "relu(add(*, *))", "explicit"]] if fused_first else []
        pats += [["b0", "add(*, *)", "explicit"], ["b0", "relu(*)", "explicit"]]
        if not fused_first:
            pats += [["b0", "relu(add(*, *))", "explicit"]]
        g = chain(["add", "relu"])
        g["nodes"][0]["inputs"] = [{"input": "x"}, {"input": "x"}]
        case = {"name": name, "graph": g, "epsilon": eps,
                "backends": [["b0", "op_kernel_library"]], "patterns": pats,
                "profiles": {"b0": profile("b0", {"add": 0.1, "relu": 0.2})}}
        cases.append(case)
    # the same near tie deep inside a longer chain (rounding at the magnitude
    # of a partial state, not of the total)
    ops = ["add", "relu"] * 6
    g = chain(ops)
    for nd in g["nodes"]:
        if nd["op"] == "add":
            nd["inputs"] = nd["inputs"] + [{"input": "x"}]
    cases.append({"name": "chain_near_ties", "graph": g, "epsilon": 0.0,
                  "backends": [["b0", "op_kernel_library"]],
                  "patterns": [["b0", "relu(add(*, *))", "explicit"], ["b0", "add(*, *)", "explicit"],
                               ["b0", "relu(*)", "explicit"]],
                  "profiles": {"b0": profile("b0", {"add": 0.1, "relu": 0.2})}})
    for case in cases:
        g = ref_graph_from_json(case["graph"])
        reg, meas = ref_registry(case)
        case["dp"] = record_dp(g, reg, meas, case["epsilon"])
        print(case["name"], case["dp"])
    with open(os.path.join(HERE, "rounding.json"), "w") as fh:
        json.dump(cases, fh, indent=1)


if __name__ == "__main__":
    main()
