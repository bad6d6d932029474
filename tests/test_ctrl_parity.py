"""Control-op strategies vs the reference's answers on the criterion-3 query set.

Goldens: every (source, target) pair with order[source] < order[target], lb
in (1, 2, 3, 5), ub in (lb, lb+2, 10) on 17 graphs (reference
test_acceptance.py:99-139), plus fallback_control on all ordered pairs.
"""

from paper_1807_02037_b200 import CtrlQuery, chain_rule, direct_order, fallback_control, graph_from_dict, topo_order
from paper_1807_02037_b200.control import CtrlIndex


def test_strategies_match_reference(ctrl_cases):
    checked = 0
    for case in ctrl_cases:
        g = graph_from_dict(case["graph"])
        order = topo_order(g)
        idx = CtrlIndex(g, order)
        for source, target, lb, ub, want_direct, want_chain in case["queries"]:
            q = CtrlQuery(source=source, target=target, lb=lb, ub=ub)
            assert idx.direct_order(q) == want_direct, (case["name"], source, target, lb, ub)
            assert idx.chain_rule(q) == want_chain, (case["name"], source, target, lb, ub)
            checked += 1
        for source, target, want in case["fallback"]:
            assert idx.fallback(source, target) == want
    assert checked > 5000


def test_public_functions_agree_with_index(ctrl_cases):
    case = ctrl_cases[1]
    g = graph_from_dict(case["graph"])
    order = topo_order(g)
    for source, target, lb, ub, want_direct, want_chain in case["queries"][:200]:
        q = CtrlQuery(source, target, lb, ub)
        assert direct_order(g, order, q) == want_direct
        assert chain_rule(g, order, q) == want_chain
    for source, target, want in case["fallback"][:50]:
        assert fallback_control(g, order, source, target) == want
