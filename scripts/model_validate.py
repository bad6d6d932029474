"""Does the calibrated model (calibrate.py) rank swap configurations like the GPU does?

ResNet-50 (or --arch), 16 GiB budget: B0 by bisection, one plain step at B0 timed per
node (node_costs), then for each candidate RewriteConfig at the target batch: the
model's predicted step time and activation peak, and the measured step time
(static plan, a few replayed steps).  Prints one JSON object with both columns and
the rank correlation.

Usage: python scripts/model_validate.py [--factor 2.0] [--lbs 1,2,3,5,8] [--ntensors -1,80]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GIB = 1 << 30


def spearman(a, b):
    ra = {v: i for i, v in enumerate(sorted(range(len(a)), key=lambda k: a[k]))}
    rb = {v: i for i, v in enumerate(sorted(range(len(b)), key=lambda k: b[k]))}
    n = len(a)
    if n < 2:
        return None
    d2 = sum((ra[k] - rb[k]) ** 2 for k in range(n))
    return 1 - 6 * d2 / (n * (n * n - 1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arch", default="resnet50")
    ap.add_argument("--budget-gib", type=float, default=16.0)
    ap.add_argument("--factor", type=float, default=2.0)
    ap.add_argument("--lbs", default="1,2,3,5,8")
    ap.add_argument("--ntensors", default="-1")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--b0", type=int, default=0)
    a = ap.parse_args()

    import torch
    import torchvision
    from paper_1807_02037_b200 import RewriteConfig, runtime as rt
    from paper_1807_02037_b200.torch_lms import LMS
    from bench import measure_host_link, is_oom

    budget = int(a.budget_gib * GIB)
    ctx = rt.Context(device=0, device_reserve=budget, host_chunk=4 * GIB, timing=True)
    rt.install_allocator(ctx)
    dev = torch.device("cuda", 0)
    link = measure_host_link(torch, dev)
    torch.backends.cudnn.benchmark = False
    torch.manual_seed(0)
    model = getattr(torchvision.models, a.arch)().to(dev)
    opt = torch.optim.SGD(model.parameters(), lr=0.1, momentum=0.9)
    lf = torch.nn.functional.cross_entropy

    def batch(n, seed=0):
        g = torch.Generator(device=dev).manual_seed(seed)
        return (torch.randn(n, 3, 224, 224, device=dev, generator=g),
                torch.randint(0, 1000, (n,), device=dev, generator=g))

    def fits(n):
        try:
            x, y = batch(n)
            for _ in range(2):
                opt.zero_grad(set_to_none=True)
                lf(model(x), y).backward()
                opt.step()
            torch.cuda.synchronize()
            return True
        except RuntimeError as e:
            if not is_oom(e):
                raise
            return False
        finally:
            opt.zero_grad(set_to_none=True)
            torch.cuda.synchronize()
            ctx.synchronize()

    b0 = a.b0
    if not b0:
        lo, hi = 0, 16
        while fits(hi):
            lo, hi = hi, hi * 2
        while hi - lo > 1:
            mid = (lo + hi) // 2
            lo, hi = (mid, hi) if fits(mid) else (lo, mid)
        b0 = lo
    x0, y0 = batch(b0)
    lms = LMS(model, lf, opt, RewriteConfig(), ctx, codec="auto", min_swap_bytes=64 << 10)
    lms.capture(*batch(4))
    lm = lms.link_model(link)
    bs = int(math.ceil(a.factor * b0))
    cfgs = [RewriteConfig(lb=lb, ub=max(10000, lb), n_tensors=n, fuse_swapins=True, swapin_fuse_distance=12)
            for lb in map(int, a.lbs.split(",")) for n in map(int, a.ntensors.split(","))]
    # one plain step at B0 timed per node -> costs scaled to bs -> each config predicted
    ranked = lms.plan_by_model(x0, y0, cfgs, bs, lm, budget)
    costs, fixed = lms.model_costs, lms.model_fixed_bytes
    del x0, y0
    xs, ys = batch(bs, seed=7)
    rows = []
    for cfg, pred, fit in ranked:
        lms.replan(cfg)
        ms = None
        try:
            for _ in range(3):
                lms.step(xs, ys)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.steps):
                lms.step(xs, ys)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
        except RuntimeError as e:
            if not is_oom(e):
                raise
            opt.zero_grad(set_to_none=True)
            torch.cuda.synchronize()
            ctx.synchronize()
        rows.append({"lb": cfg.lb, "n_tensors": cfg.n_tensors, "predicted_ms": round(pred["makespan"] * 1e3, 1),
                     "predicted_peak_gib": round((pred["peak_device_bytes"] + fixed) / GIB, 2),
                     "predicted_fits": fit, "predicted_alloc_stall_ms": round(pred["alloc_stall"] * 1e3, 1),
                     "measured_ms": None if ms is None else round(ms, 1)})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    both = [r for r in rows if r["measured_ms"] is not None]
    out = {"arch": a.arch, "b0": b0, "batch": bs, "budget_gib": a.budget_gib,
           "plain_step_ms_at_b0": round((costs["_forward_total"] + costs["_backward_total"] +
                                         costs["_optimizer_total"]) * 1e3, 1),
           "fixed_gib": round(fixed / GIB, 2), "link": link, "rows": rows,
           "spearman_predicted_vs_measured": spearman([r["predicted_ms"] for r in both],
                                                      [r["measured_ms"] for r in both]),
           "fit_agreement": sum((r["measured_ms"] is not None) == r["predicted_fits"] for r in rows) / len(rows)}
    if both:
        best_pred = min(both, key=lambda r: r["predicted_ms"])
        best_meas = min(both, key=lambda r: r["measured_ms"])
        out["model_pick"] = best_pred
        out["measured_best"] = best_meas
        out["model_pick_vs_best"] = round(best_pred["measured_ms"] / best_meas["measured_ms"], 3)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
