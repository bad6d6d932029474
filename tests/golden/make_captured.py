"""Golden rewrites of CAPTURED model graphs, produced by the REFERENCE rewrite.

Run in the build container (the read-only reference is importable there):

    python tests/golden/make_captured.py

The graphs are what ``torch_lms.capture_graph`` records for the BASELINE
workloads on CPU (the same capture settings ``bench.py`` uses: ResNet-50 at
batch 4, 224^2; the 3D U-Net at batch 1, 32^3; ResNet-152 at batch 1), stored
as graph dicts.  For each, the reference ``swapgraph.rewrite`` runs over a
grid of configurations — including the headline bench's (lb 1, chain_rule,
fuse_swapins at distance 12), the paper's 3DUnet setting (swap_branches,
threshold 20, lb 1) and the ResNet-152 autotune pick (lb 8) — and the sha256
of its ``dumps`` plus its report dict are written to ``captured_cases.json.gz``.
Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import swapgraph as R  # noqa: E402  (the reference)

from paper_1807_02037_b200.serialize import dumps as our_dumps, graph_to_dict  # noqa: E402

sys.path.insert(0, HERE)
from capture_recipe import capture  # noqa: E402


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def cfg_dict(cfg) -> dict:
    return {k: sorted(v) if isinstance(v, frozenset) else v for k, v in cfg.__dict__.items()}


def grid(name):
    bench = dict(lb=1, ctrld_strategy="chain_rule", fuse_swapins=True, swapin_fuse_distance=12)
    cfgs = [R.RewriteConfig(), R.RewriteConfig(**bench), R.RewriteConfig(lb=3, ctrld_strategy="direct_order")]
    if name == "resnet152":
        return [R.RewriteConfig(lb=8), R.RewriteConfig(**bench)]
    cfgs += [R.RewriteConfig(n_tensors=40, **bench),
             R.RewriteConfig(lb=8),
             R.RewriteConfig(fuse_swapins=True, swapin_fuse_distance=0),
             R.RewriteConfig(swap_branches=True, branch_threshold=20, lb=1),
             R.RewriteConfig(swap_branches=True, branch_threshold=5, ctrld_strategy="direct_order", lb=2),
             R.RewriteConfig(excl_types=frozenset({"Relu"}), lb=2)]
    return cfgs


def main():
    out = []
    for name in ("resnet50", "unet3d", "resnet152"):
        g_ours = capture(name)
        d = graph_to_dict(g_ours)
        g = R.graph_from_dict(d)
        assert R.dumps(g) == our_dumps(g_ours)
        results = []
        for cfg in grid(name):
            t0 = time.perf_counter()
            o, rep = R.rewrite(g, cfg)
            results.append({"cfg": cfg_dict(cfg), "sha256": sha(R.dumps(o)), "report": rep.to_dict(),
                            "reference_seconds": round(time.perf_counter() - t0, 2)})
            print(name, results[-1]["cfg"]["lb"], rep.tensors_swapped, results[-1]["reference_seconds"], "s",
                  flush=True)
        out.append({"name": name, "graph": d, "graph_sha256": sha(R.dumps(g)), "results": results})
    path = os.path.join(HERE, "captured_cases.json.gz")
    with gzip.open(path, "wt") as fh:
        json.dump(out, fh, separators=(",", ":"), sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
