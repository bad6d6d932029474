"""Which part of a swapped-vs-plain difference is swapping and which is cuDNN?

Runs tests/_parity_worker.py for plain (twice) and swapped runs at a large and
a tight budget, and prints per-tensor relative errors against the first plain run.
Usage: python scripts/parity_probe.py unet3d [tight_gib]
"""
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W = os.path.join(ROOT, "tests", "_parity_worker.py")
model = sys.argv[1] if len(sys.argv) > 1 else "unet3d"
tight = sys.argv[2] if len(sys.argv) > 2 else "1.72"
env = dict(os.environ, CUDNN_CONV_WSCAP_DBG=os.environ.get("CUDNN_CONV_WSCAP_DBG", "128"))
extra = sys.argv[3:]   # e.g. --branches
runs = {"plainA": ["plain", "--budget-gib", "40"], "plainB": ["plain", "--budget-gib", "40"],
        "swap40": ["swap", "--budget-gib", "40", *extra],
        "swaptight": ["swap", "--budget-gib", tight, "--page-mb", "8", *extra]}
res = {}
for name, args in runs.items():
    out = f"/tmp/probe_{name}.pt"
    r = subprocess.run([sys.executable, W, args[0], model, out, *args[1:], "--steps", "3"], env=env,
                       capture_output=True, text=True)
    print(name, r.returncode, r.stdout.strip()[-300:], r.stderr.strip()[-500:])
    res[name] = torch.load(out)
ref = res["plainA"]
for name, d in res.items():
    worst = []
    for k, v in ref["state"].items():
        if v.is_floating_point():
            e = float((d["state"][k].double() - v.double()).norm() / max(float(v.double().norm()), 1e-30))
            worst.append((e, k))
    worst.sort(reverse=True)
    print(name, "losses", [float(x) for x in d["losses"]], "bit-equal losses",
          all(torch.equal(a, b) for a, b in zip(d["losses"], ref["losses"])), "worst", worst[:3])
