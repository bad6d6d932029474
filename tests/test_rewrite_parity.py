"""Bit-exact parity of the rewrite API against golden vectors from the reference.

The goldens (tests/golden/make_golden.py) hold, per input graph and config,
the sha256 of the reference's ``dumps(rewrite(g, cfg))`` and its
``RewriteReport.to_dict()`` (or its exception text).  Acceptance rule:
SURVEY.md §8(c)(1) — byte-identical canonical JSON and identical reports.
"""

import hashlib

import pytest

from paper_1807_02037_b200 import (
    RewriteConfig,
    dumps,
    graph_from_dict,
    rewrite,
    topo_order,
)
from paper_1807_02037_b200 import generate as G


def _sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


def _cfg(d):
    kw = dict(d)
    for k in ("optimizer_scopes", "starting_op_names", "excl_scopes", "incl_scopes",
              "excl_types", "incl_types"):
        kw[k] = frozenset(kw[k])
    return RewriteConfig(**kw)


def test_inputs_roundtrip_bytes(rewrite_cases):
    for case in rewrite_cases:
        g = graph_from_dict(case["graph"])
        assert _sha(dumps(g)) == case["input_dumps_sha256"], case["name"]


def test_topo_order_matches(rewrite_cases):
    for case in rewrite_cases:
        if "order" not in case:
            continue
        g = graph_from_dict(case["graph"])
        want = {int(k): v for k, v in case["order"].items()}
        assert topo_order(g) == want, case["name"]


def test_rewrite_bit_exact(rewrite_cases):
    checked = errors = 0
    for case in rewrite_cases:
        g = graph_from_dict(case["graph"])
        for res in case["results"]:
            cfg = _cfg(res["cfg"])
            if "error" in res:
                with pytest.raises(Exception) as info:
                    rewrite(g, cfg)
                got = f"{type(info.value).__name__}: {info.value}"
                assert got == res["error"], (case["name"], res["cfg"])
                errors += 1
                continue
            out, rep = rewrite(g, cfg)
            text = dumps(out)
            if "dumps" in res:
                assert text == res["dumps"], (case["name"], res["cfg"])
            assert _sha(text) == res["sha256"], (case["name"], res["cfg"])
            assert rep.to_dict() == res["report"], (case["name"], res["cfg"])
            checked += 1
    assert checked > 5000
    assert errors > 0


@pytest.mark.parametrize("builder,args", [
    (G.chain, (1,)), (G.chain, (20,)), (G.chain, (100,)), (G.branchy, (8,)), (G.branchy, (20,)),
    (G.unet, (3,)), (G.unet, (4, 8 << 20)), (G.resnet_like, (4,)), (G.resnet_like, (16,)),
    (G.chain, (317,)), (G.resnet_like, (50,)),
])
def test_generators_identical(rewrite_cases, builder, args):
    names = {"chain": "chain", "branchy": "branchy", "unet": "unet", "resnet_like": "resnet_like"}
    label = f"gen:{names[builder.__name__]}({args[0]}" + (",8MiB)" if len(args) > 1 else ")")
    case = next(c for c in rewrite_cases if c["name"] == label)
    assert _sha(dumps(builder(*args))) == case["input_dumps_sha256"]


def test_fig5_golden(rewrite_cases):
    """Acceptance criterion 1 (reference test_acceptance.py:36-67)."""
    from paper_1807_02037_b200 import EdgeAction, EdgeRec, lifetime, validate
    case = next(c for c in rewrite_cases if c["name"] == "fixture:hot_fanout_graph")
    g = graph_from_dict(case["graph"])
    order = topo_order(g)
    assert (order[10], order[34], order[33], order[25]) == (10, 11, 18, 25)
    assert lifetime(g, order, 10) == 15
    out, rep = rewrite(g, RewriteConfig(swap_branches=True, branch_threshold=5,
                                        ctrld_strategy="direct_order", lb=5, ub=9))
    assert rep.edges_rewritten == [(10, 25, 10), (10, 33, 10)]
    assert EdgeRec(10, 34, EdgeAction.READ, 10) in out.edges
    assert (rep.tensors_swapped, rep.swap_outs_added, rep.swap_ins_added,
            rep.control_edges_added) == (1, 1, 2, 2)
    ctrl = sorted((e.src, e.dst) for e in out.edges if e.action is EdgeAction.CONTROL)
    assert ctrl == [(20, 36), (28, 38)]
    assert validate(out) == []
