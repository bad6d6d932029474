"""Planning cost of the rewrite: ours vs the reference, same graphs.

Run in the build container (the reference is importable read-only there):
    python scripts/rewrite_speed.py [--ref] > profiles/r01/rewrite_speed.json
Both outputs are checked byte-identical (dumps) on every graph timed.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", action="store_true", help="also time the reference (needs /root/reference)")
    ap.add_argument("--sizes", default="100,317,1000")
    a = ap.parse_args()
    import paper_1807_02037_b200 as ours
    ref = None
    if a.ref:
        sys.path.insert(0, "/root/reference/pkg/src")
        import swapgraph as ref  # noqa: F401  (read-only reference, timing only)
    rows = []
    for n in [int(x) for x in a.sizes.split(",")]:
        for strat in ("chain_rule", "direct_order"):
            g = ours.chain(n)
            t = time.perf_counter()
            out, rep = ours.rewrite(g, ours.RewriteConfig(ctrld_strategy=strat))
            dt = time.perf_counter() - t
            row = {"graph": f"chain({n})", "strategy": strat, "nodes": len(g.nodes),
                   "tensors_swapped": rep.tensors_swapped, "ours_s": round(dt, 4)}
            if ref is not None:
                rg = ref.chain(n)
                t = time.perf_counter()
                rout, rrep = ref.rewrite(rg, ref.RewriteConfig(ctrld_strategy=strat))
                row["reference_s"] = round(time.perf_counter() - t, 3)
                row["identical"] = ref.dumps(rout) == ours.dumps(out) and rrep.to_dict() == rep.to_dict()
                row["speedup"] = round(row["reference_s"] / max(dt, 1e-9), 1)
            rows.append(row)
            print(json.dumps(row), file=sys.stderr)
    print(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
