"""The CPU oracle (oracle/interp_oracle.py) pinned against the reference's outputs.

Golden vectors: reference ``interpret`` on graphgen seeds 0-39 and on the C1
ffchain, before and after rewrite (tests/golden/make_golden.py).  The oracle
uses the same float64 numpy operations in the same order, so agreement is
bit-exact.
"""

import numpy as np
import pytest

from oracle.interp_oracle import interpret as oracle_interpret
from paper_1807_02037_b200 import graph_from_dict


def _arrays(d):
    return {k: np.asarray(v, dtype=np.float64) for k, v in d.items()}


def test_oracle_matches_reference_interpret(interp_cases):
    checked = 0
    for case in interp_cases:
        g = graph_from_dict(case["graph"])
        inputs = _arrays(case["inputs"])
        got = oracle_interpret(g, inputs)
        want = _arrays(case["outputs"])
        assert got.keys() == want.keys()
        for k in want:
            assert np.array_equal(got[k], want[k]), (case["name"], k)
        for rw in case["rewritten"]:
            g2 = graph_from_dict(rw["graph"])
            got2 = oracle_interpret(g2, inputs)
            for k, v in _arrays(rw["outputs"]).items():
                assert np.array_equal(got2[k], v), (case["name"], rw["cfg"], k)
                assert np.array_equal(got2[k], want[k])  # swapping preserves semantics
            checked += 1
    assert checked >= 100


def test_oracle_errors_like_reference():
    from paper_1807_02037_b200 import CompGraph, EdgeAction, EdgeRec, TensorSpec, compute_node, variable_node
    g = CompGraph([variable_node(0, "x"), compute_node(1, "frob")],
                  [EdgeRec(0, 1, EdgeAction.READ, 0)],
                  [TensorSpec(0, 0, 8), TensorSpec(1, 1, 8)])
    with pytest.raises(ValueError, match="unsupported op 'frob'"):
        oracle_interpret(g, {"x": np.ones((2, 2))})
    with pytest.raises(ValueError, match="unbound"):
        oracle_interpret(g, {})
