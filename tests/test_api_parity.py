"""Standalone public pass functions against the reference's own answers.

Golden file ``api_cases.json.gz`` (tests/golden/make_golden.py) holds what the
reference returned for:

* ``insert_swap_pair(g, edge)`` on the fixtures/generators/graphgen seeds,
  candidate edges plus invalid ones (ref tests/test_rewriter.py:191-213:
  ids max+1/+2, names, host placement, rewired edges — here the whole output
  graph by ``dumps`` sha256, and the error text for bad edges);
* ``attach_control(g, ctrl, swap_in)`` on rewritten graphs with their control
  edges stripped, over a spread of (ctrl, swap_in) pairs including unknown
  ids, parameterized targets and cycle-closing edges (ref control.py:158-169);
* ``free_step_oracle`` for every tensor of every graph, plain and rewritten
  (ref sim.py:479-508);
* the reference package's ``__all__`` (ref __init__.py:60-115).
"""

import hashlib

import pytest

import paper_1807_02037_b200 as P
from paper_1807_02037_b200 import (
    EdgeAction,
    EdgeRec,
    attach_control,
    dumps,
    free_step_oracle,
    graph_from_dict,
    insert_swap_pair,
)

from conftest import load_golden


@pytest.fixture(scope="module")
def api():
    return load_golden("api_cases.json.gz")


def _sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


def test_facade_is_superset_of_reference_all(api):
    ref = set(api["reference_all"])
    assert len(ref) == 54
    assert ref <= set(P.__all__)
    missing = [n for n in sorted(ref) if not hasattr(P, n)]
    assert missing == []


def test_insert_swap_pair_matches_reference(api):
    graphs = {k: graph_from_dict(v) for k, v in api["graphs"].items()}
    n_ok = n_err = 0
    for case in api["insert_swap_pair"]:
        g = graphs[case["graph"]]
        src, dst, action, tensor = case["edge"]
        e = EdgeRec(src, dst, EdgeAction(action), tensor)
        if "error" in case:
            with pytest.raises(Exception) as info:
                insert_swap_pair(g, e)
            assert f"{type(info.value).__name__}: {info.value}" == case["error"]
            n_err += 1
            continue
        out, so, si = insert_swap_pair(g, e)
        assert (so, si) == (case["so"], case["si"])
        assert _sha(dumps(out)) == case["sha256"], (case["graph"], case["edge"])
        n_ok += 1
    assert n_ok >= 100 and n_err >= 20


def test_insert_swap_pair_structure():
    # ref tests/test_rewriter.py:191-213 on its three_op_chain fixture shape
    from paper_1807_02037_b200 import HOST, NodeKind, chain
    g = chain(2)
    e = next(x for x in g.edges if x.action is EdgeAction.READ
             and g.node_by_id[x.dst].name.startswith("bwd"))
    out, so_id, si_id = insert_swap_pair(g, e)
    so, si = out.node_by_id[so_id], out.node_by_id[si_id]
    assert (so_id, si_id) == (g.max_node_id() + 1, g.max_node_id() + 2)
    assert so.kind is NodeKind.SWAP_OUT and si.kind is NodeKind.SWAP_IN
    assert so.device == HOST == si.device and so.scope == si.scope == "swap"
    assert so.name == f"swap_out_{e.tensor}_{e.dst}" and si.name == f"swap_in_{e.tensor}_{e.dst}"
    assert e not in out.edges


def test_attach_control_matches_reference(api):
    graphs = {k: graph_from_dict(v) for k, v in api["graphs"].items()}
    seen = {"ok": 0, "KeyError": 0, "ValueError": 0}
    for case in api["attach_control"]:
        g = graphs[case["graph"]]
        if "error" in case:
            with pytest.raises(Exception) as info:
                attach_control(g, case["ctrl"], case["swap_in"])
            got = f"{type(info.value).__name__}: {info.value}"
            assert got == case["error"], case
            seen[type(info.value).__name__] += 1
            continue
        out = attach_control(g, case["ctrl"], case["swap_in"])
        assert _sha(dumps(out)) == case["sha256"], case
        seen["ok"] += 1
    assert seen["ok"] >= 100 and seen["KeyError"] >= 10 and seen["ValueError"] >= 50


def test_free_step_oracle_matches_reference(api):
    n = 0
    for case in api["free_step_oracle"]:
        g = graph_from_dict(case["graph"])
        order = {int(k): v for k, v in case["order"].items()}
        for tid, step in case["free_steps"].items():
            assert free_step_oracle(g, order, int(tid)) == step
            n += 1
    assert n > 800


def test_free_step_equals_order_plus_lifetime():
    # criterion 4 (ref test_acceptance.py:142-164) on the generators
    from paper_1807_02037_b200 import chain, lifetime, rewrite, RewriteConfig, topo_order, unet
    for g in (chain(12), unet(3), rewrite(chain(8), RewriteConfig())[0]):
        order = topo_order(g)
        for t in g.tensors:
            if not g.node_by_id[t.producer].parameterized:
                assert free_step_oracle(g, order, t.id) == order[t.producer] + lifetime(g, order, t.id)


def test_simulate_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    from paper_1807_02037_b200 import SimConfig, chain, simulate, topo_order
    from paper_1807_02037_b200.runtime import LmsError
    g = chain(3)
    with pytest.raises(LmsError):
        simulate(g, topo_order(g), SimConfig())
    bad = chain(3, tensor_bytes=0)
    with pytest.raises(ValueError, match="size_bytes=0"):
        simulate(bad, topo_order(bad), SimConfig())
