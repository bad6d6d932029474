"""Rewrite parity on CAPTURED model graphs (north-star rule 1 at model scale).

``captured_cases.json.gz`` (tests/golden/make_captured.py) holds the graphs
``capture_graph`` records for ResNet-50, the 3D U-Net and ResNet-152 with the
bench's capture settings, and what the REFERENCE ``rewrite`` produced on them
over a grid of configurations (the headline bench's, the paper's 3DUnet
swap_branches setting, the ResNet-152 autotune lb 8, direct_order, n_tensors
caps, fusion distances, type exclusion).  Our rewrite must give the same
``dumps`` byte for byte and the same report.
"""

import hashlib

import pytest

from paper_1807_02037_b200 import RewriteConfig, dumps, graph_from_dict, rewrite

from conftest import load_golden


def _sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


def _cfg(d):
    kw = {k: frozenset(v) if isinstance(v, list) else v for k, v in d.items()}
    return RewriteConfig(**kw)


@pytest.fixture(scope="module")
def captured():
    return load_golden("captured_cases.json.gz")


def test_captured_graphs_rewrite_like_the_reference(captured):
    n = 0
    for case in captured:
        g = graph_from_dict(case["graph"])
        assert _sha(dumps(g)) == case["graph_sha256"]
        for r in case["results"]:
            out, rep = rewrite(g, _cfg(r["cfg"]))
            assert _sha(dumps(out)) == r["sha256"], (case["name"], r["cfg"])
            assert rep.to_dict() == r["report"], (case["name"], r["cfg"])
            n += 1
    assert {c["name"] for c in captured} == {"resnet50", "unet3d", "resnet152"}
    assert n >= 20


def test_capture_is_deterministic(captured):
    """Capturing the 3D U-Net again gives the stored graph byte for byte."""
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    torch = pytest.importorskip("torch")
    pytest.importorskip("torchvision")
    case = next(c for c in captured if c["name"] == "unet3d")
    from capture_recipe import capture   # the generator's capture recipe
    g = capture("unet3d")
    assert _sha(dumps(g)) == case["graph_sha256"]
    del torch
