"""Measurer bookkeeping of the REFERENCE DP (tensorplace/dp.py:71-179 calls
SimMeasurer.measure_kernel once per candidate; tensorplace/cost.py:248-263):
counters of a cold and a warm optimize run on one measurer, and the cache
contents after the cold run.

    python tests/golden/make_measurer_golden.py   (build container only)
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import ref, ref_graph_from_json, ref_registry  # noqa: E402


def main():
    out = []
    for suite, names in (("fixtures", None), ("models", ["resnet50", "bert_base"]),
                         ("dp_random", None), ("dp_ties", None)):
        with open(os.path.join(HERE, f"{suite}.json")) as fh:
            cases = json.load(fh)
        picked = [c for c in cases if names is None or c["name"] in names]
        if names is None:
            picked = picked[:8]
        for case in picked:
            if "error" in case["dp"]:
                continue
            g = ref_graph_from_json(case["graph"])
            reg, meas = ref_registry(dict(case))
            runs = []
            for _ in range(2):
                res = ref.optimize(g, reg, meas, case["epsilon"], max_states=200_000)
                runs.append({"measure_calls": res.stats.measure_calls,
                             "cache_hits": res.stats.cache_hits,
                             "computations": res.stats.computations})
                if len(runs) == 1:
                    items = sorted(meas.cache.items())
            out.append({"suite": suite, "name": case["name"], "runs": runs,
                        "cache_size": len(items),
                        "cache_sha256": hashlib.sha256(json.dumps(items).encode()).hexdigest(),
                        "counters": {"calls": meas.calls, "cache_hits": meas.cache_hits,
                                     "computations": meas.computations}})
            print(out[-1]["name"], runs, len(items))
    with open(os.path.join(HERE, "measurer.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
