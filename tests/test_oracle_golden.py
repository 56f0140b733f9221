"""The CPU oracle against the reference's own outputs (tests/golden)."""

import numpy as np
import pytest

from conftest import golden
from oracle import OracleCase, window_safe

SUITES = ["fixtures", "dp_random", "dp_ties", "dp_large", "es_random", "models"]


def _cases():
    for s in SUITES:
        for c in golden(s):
            yield pytest.param(c, id=c["name"])


@pytest.mark.parametrize("case", list(_cases()))
def test_oracle_reproduces_reference(case):
    oc = OracleCase(case)
    if "candidates" in case:
        assert oc.candidates() == case["candidates"]
    oc.price()
    exp = case["dp"]
    status, cost, kernels = oc.dp(max_states=200_000 if case["name"] in
                                  ("resnet50", "bert_base", "nasrnn") else 50_000)
    if "error" in exp:
        want = {"UncoverableGraphError": "uncoverable", "SearchLimitError": "limit"}[exp["error"]]
        assert status == want
        return
    assert status == "ok"
    assert cost == exp["cost"]
    assert kernels == exp["kernels"]
    assert oc.dp_relaxations == exp["relaxations"]
    # the independent solver (post-dominator subtrees) pins the configs the
    # reference cannot solve (tests/test_dp_pins.py); here it must return the
    # reference's own result on every case the reference solved
    s2, cost2, kernels2, regret = oc.dp_subtree()
    assert (s2, cost2, kernels2) == ("ok", exp["cost"], exp["kernels"])
    assert window_safe(cost2, regret)
    if "es" in case:
        es = case["es"]
        fit = oc.fitness(exp["kernels"], es["graph_backend"], es["genomes"])
        assert np.array_equal(fit, np.array(es["fitness"]))


def test_oracle_matcher_suite():
    from paper_2111_00655_b200.patterns import CompiledPatterns, parse_pattern
    checked = 0
    for case in golden("matcher"):
        oc = OracleCase(case)
        for text, want in case["matches"].items():
            cp = CompiledPatterns([parse_pattern(text)], [0])
            mt = oc.match_all(cp)
            got = []
            for m in range(mt["n"]):
                root = oc.ids[int(np.searchsorted(mt["group_ptr"], m, side="right") - 1)]
                mem = sorted(oc.ids[x] for x in mt["members"][mt["mem_ptr"][m]:mt["mem_ptr"][m + 1]])
                binds = mt["binds"][mt["bind_ptr"][m]:mt["bind_ptr"][m + 1]]
                binding = sorted((list(cp.paths[0][i]), oc.ids[x]) for i, x in enumerate(binds))
                got.append([root, mem, [[p, x] for p, x in binding]])
            assert got == want, (case["name"], text)
            checked += 1
    assert checked >= 300
