"""Swap overhead vs oversubscription (BASELINE: "<=25 % step-time overhead versus
no-swap"): ResNet-50 under the 16 GiB budget at batch = f x B0 for several f, each
with the fewest swapped tensors that fit (bench.py --search), reported per image
against the no-swap step at B0.

Usage: python scripts/overhead_curve.py [--factors 1.25,1.5,2,3,4.7] [--b0 193]
Writes gpurun_out/overhead_<arch>.json and .md.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from frontier import ROOT, run  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arch", default="resnet50")
    ap.add_argument("--factors", default="1.25,1.5,2,3,4.7")
    ap.add_argument("--b0", type=int, default=0)
    ap.add_argument("--budget-gib", type=float, default=16.0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--search", type=int, default=6)
    ap.add_argument("--timeout", type=int, default=900)
    ap.add_argument("--extra", default="", help="more bench.py arguments, e.g. '--tune-windows 1'")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    common = ["--arch", a.arch, "--budget-gib", str(a.budget_gib), "--steps", str(a.steps),
              "--warmup", "3", "--cpu-baseline", "0", "--same-batch", "0", "--search", str(a.search)]
    if a.b0:
        common += ["--b0", str(a.b0)]
    common += a.extra.split()
    rows = []
    for f in [float(x) for x in a.factors.split(",")]:
        r = run(common + ["--factor", str(f)], a.timeout)
        r["factor"] = f
        rows.append(r)
        print(json.dumps({k: r.get(k) for k in ("factor", "value", "ms_per_step", "error")}), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"overhead_{a.arch}{a.tag}.json"), "w") as fh:
        json.dump(rows, fh)
    lines = [f"# {a.arch}: swap overhead vs oversubscription under {a.budget_gib:g} GiB {a.extra}", "",
             "overhead = (no-swap img/s at B0) / (swapped img/s at f x B0) - 1, per image", "",
             "| f | batch | tensors swapped | img/s | ms/step | D2H GB | overhead | tuner trial ms | timed / trial |",
             "|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        if "error" in r:
            lines.append(f"| {r['factor']} | error: {r['error']} | | | | | |")
            continue
        s, ns = r["swap"], r["no_swap"]
        ov = ns["img_s"] / r["value"] - 1
        tw = s.get("tune_windows") or {}
        trial = tw.get("final_ms") or (tw.get("trials") or {}).get(str(tw.get("moved"))) or tw.get("base_ms")
        ratio = f"{r['ms_per_step'] / trial:.3f}" if trial else "-"
        lines.append(f"| {r['factor']} | {r['config']['per_gpu_batch']} | {s['tensors_swapped']} | {r['value']} | "
                     f"{r['ms_per_step']} | {s['d2h_bytes_per_step'] / 1e9:.1f} | {ov:+.1%} | "
                     f"{round(trial, 1) if trial else '-'} | {ratio} |")
    md = "\n".join(lines) + "\n"
    with open(os.path.join(ROOT, "gpurun_out", f"overhead_{a.arch}{a.tag}.md"), "w") as fh:
        fh.write(md)
    print(md)


if __name__ == "__main__":
    main()
