"""Overlap-vs-overhead frontier (BASELINE configs[4]): lb/ub and swap-set sweeps at an
oversubscribed batch, one bench.py run per point, summarised as a table.

Usage: python scripts/frontier.py --arch resnet152 --factor 3 [--lbs 1,2,3,5,8] [--ns 0,-1]
Writes gpurun_out/frontier_<arch>.json and .md.  The paper's trade-off:
a larger lb starts swap-ins earlier (less stall, more memory); fewer swapped tensors cut
traffic but raise the peak.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args_list, timeout):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py")] + args_list
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    line = next((ln for ln in reversed(p.stdout.strip().splitlines()) if ln.startswith("{")), None)
    if p.returncode != 0 or line is None:
        return {"error": (p.stderr.strip().splitlines() or ["?"])[-1][:200], "args": args_list}
    return json.loads(line)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arch", default="resnet152")
    ap.add_argument("--factor", type=float, default=3.0)
    ap.add_argument("--budget-gib", type=float, default=16.0)
    ap.add_argument("--lbs", default="1,2,3,5,8")
    ap.add_argument("--ns", default="0")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--timeout", type=int, default=900)
    a = ap.parse_args()
    common = ["--arch", a.arch, "--factor", str(a.factor), "--budget-gib", str(a.budget_gib),
              "--steps", str(a.steps), "--warmup", "3", "--cpu-baseline", "0"]
    first = run(common + ["--lb", "1"], a.timeout)
    rows = [first]
    b0 = first.get("config", {}).get("no_swap_max_batch")
    if b0:
        common += ["--b0", str(b0)]
    for lb in [int(x) for x in a.lbs.split(",")]:
        for n in [int(x) for x in a.ns.split(",")]:
            if lb == 1 and n == 0:
                continue
            rows.append(run(common + ["--lb", str(lb), "--n-tensors", str(n)], a.timeout))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"frontier_{a.arch}.json"), "w") as fh:
        json.dump(rows, fh)
    lines = [f"# {a.arch} frontier: factor {a.factor} x B0 under {a.budget_gib:g} GiB", "",
             "| lb | tensors swapped | batch | samples/s | ms/step | D2H GB | H2D GB | peak GiB | stall ms/step |",
             "|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        if "error" in r:
            lines.append(f"| {r['args']} | error: {r['error']} | | | | | | | |")
            continue
        c, s = r["config"], r["swap"]
        lines.append(f"| {c['rewrite']['lb']} | {s['tensors_swapped']} | {c['per_gpu_batch']} | {r['value']} | "
                     f"{r['ms_per_step']} | {s['d2h_bytes_per_step'] / 1e9:.1f} | {s['h2d_bytes_per_step'] / 1e9:.1f} | "
                     f"{s['device_peak_bytes'] / 2**30:.2f} | {s['swap_wait_ms_per_step']} |")
    if b0:
        lines.insert(1, f"no-swap max batch B0 = {b0}, no-swap {first['no_swap']['img_s']} samples/s")
    md = "\n".join(lines) + "\n"
    with open(os.path.join(ROOT, "gpurun_out", f"frontier_{a.arch}.md"), "w") as fh:
        fh.write(md)
    print(md)


if __name__ == "__main__":
    main()
