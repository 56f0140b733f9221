"""Near-tie cases (tests/golden/rounding.json, solved by the reference):
an alternative partition within one ulp of the optimum, where the
reference's rounded state comparisons (tensorplace/dp.py:128-147) and the
device's exact ones can disagree.  The device must not silently return a
placement the reference would not: uncertified results raise
RoundingWindowError (carrying the exact optimum)."""

import math

import pytest

from conftest import build_case, golden, kernels_of
from oracle import OracleCase, window_safe

CASES = golden("rounding")


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_reproduces_reference_and_flags_the_window(case):
    oc = OracleCase(case)
    oc.price()
    status, cost, kernels = oc.dp()
    assert (status, cost, kernels) == ("ok", case["dp"]["cost"], case["dp"]["kernels"])
    s2, c2, k2, regret = oc.dp_subtree()
    assert s2 == "ok"
    if case["epsilon"] > 0:
        assert window_safe(c2, regret) and (c2, k2) == (cost, kernels)
    else:
        # exact optimum: the two singletons (0.1 + 0.2 < round(0.1 + 0.2))
        assert not window_safe(c2, regret)
        assert all(len(nodes) == 1 for _, _, nodes in k2)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_device_refuses_uncertified_ties(gpu, case):
    import paper_2111_00655_b200 as tp
    g, reg, meas = build_case(case)
    if case["epsilon"] > 0:
        res = tp.optimize(g, reg, meas, case["epsilon"])
        assert res.device["rounding_window_safe"]
        assert (res.cost_ms, kernels_of(res.placement)) == (case["dp"]["cost"], case["dp"]["kernels"])
        return
    with pytest.raises(tp.RoundingWindowError) as info:
        tp.optimize(g, reg, meas, case["epsilon"])
    exact = info.value.result
    assert isinstance(info.value, tp.SearchLimitError)
    assert not exact.device["rounding_window_safe"]
    res = tp.optimize(g, reg, meas, case["epsilon"], rounding="exact")
    assert kernels_of(res.placement) == kernels_of(exact.placement)
    assert all(len(a.nodes) == 1 for a in res.placement.assignments)
    # the rounded total is the reference's (the partitions differ, the double does not)
    assert res.cost_ms == case["dp"]["cost"] or math.isclose(res.cost_ms, case["dp"]["cost"])
