"""Back-to-back swapped steps (no host sync between them), as bench.py times them.

Usage: python scripts/backtoback.py --batch 908 --steps 8 [--codec auto] [--e2e]
Prints per-step device time (CUDA events) and the host-side pool counters per step.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=908)
    ap.add_argument("--budget-gib", type=float, default=16.0)
    ap.add_argument("--codec", default="auto")
    ap.add_argument("--tf32", action="store_true")
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--e2e", action="store_true")
    ap.add_argument("--no-plan", action="store_true")
    ap.add_argument("--no-trim", action="store_true")
    ap.add_argument("--refine", default="2", help="comma list of steps that refine the plan")
    ap.add_argument("--n-tensors", type=int, default=-1)
    ap.add_argument("--lb", type=int, default=1)
    ap.add_argument("--far-lb", type=int, default=0)
    ap.add_argument("--far-frac", type=float, default=0.0)
    ap.add_argument("--pre", default="", help="comma list of n_tensors: 2 dynamic steps each before the run "
                                            "(what bench.py's fit probes do)")
    args = ap.parse_args()

    import torch
    import torchvision
    from paper_1807_02037_b200 import RewriteConfig, runtime as rt
    from paper_1807_02037_b200.torch_lms import LMS

    ctx = rt.Context(device=0, device_reserve=int(args.budget_gib * (1 << 30)), host_chunk=4 << 30, timing=True)
    rt.install_allocator(ctx)
    torch.backends.cudnn.benchmark = False
    # strict fp32 like bench.py (the BASELINE config); --tf32 lets cuDNN use TF32 tensor cores
    torch.backends.cudnn.allow_tf32 = bool(args.tf32)
    torch.backends.cuda.matmul.allow_tf32 = bool(args.tf32)
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    model = torchvision.models.resnet50().to(dev)
    opt = torch.optim.SGD(model.parameters(), lr=0.1, momentum=0.9)
    lf = torch.nn.functional.cross_entropy
    lms = LMS(model, lf, opt, RewriteConfig(fuse_swapins=True, swapin_fuse_distance=1), ctx, codec=args.codec,
              min_swap_bytes=64 << 10, static_plan=not args.no_plan)
    LMS.REFINE_STEPS = tuple(int(x) for x in args.refine.split(",") if x)
    if args.no_trim:
        ctx.trim = lambda: 0
    xc = torch.randn(4, 3, 224, 224, device=dev)
    yc = torch.randint(0, 1000, (4,), device=dev)
    lms.capture(xc, yc)
    x = torch.randn(args.batch, 3, 224, 224, device=dev)
    y = torch.randint(0, 1000, (args.batch,), device=dev)
    for n_pre in [int(v) for v in args.pre.split(",") if v]:
        lms.replan(RewriteConfig(fuse_swapins=True, swapin_fuse_distance=1, n_tensors=n_pre, lb=args.lb))
        lms.static_plan = False
        for _ in range(2):
            lms.step(x, y)
        torch.cuda.synchronize()
    lms.static_plan = not args.no_plan
    if args.far_lb:
        lms.far_cfg = RewriteConfig(fuse_swapins=True, swapin_fuse_distance=1, n_tensors=args.n_tensors,
                                    lb=args.far_lb)
        lms.far_max_fraction = args.far_frac
    lms.replan(RewriteConfig(fuse_swapins=True, swapin_fuse_distance=1, n_tensors=args.n_tensors, lb=args.lb))
    del xc, yc
    if args.e2e:
        xh, yh = x.cpu().pin_memory(), y.cpu().pin_memory()
        del x, y
    s = torch.cuda.current_stream()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    keys = ("n_reclaims", "pool_driver_ms", "alloc_wait_ms", "n_device_syncs")
    host = []
    torch.cuda.synchronize()
    evs[0].record(s)
    for i in range(args.steps):
        st0 = ctx.stats()
        if args.e2e:
            xb = xh.to(dev, non_blocking=True)
            yb = yh.to(dev, non_blocking=True)
            loss = lms.step(xb, yb)
            loss.item()
        else:
            lms.step(x, y)
        evs[i + 1].record(s)
        st1 = ctx.stats()
        host.append({k: round(st1[k] - st0[k], 1) for k in keys})
    torch.cuda.synchronize()
    out = []
    for i in range(args.steps):
        out.append({"step": i, "ms": round(evs[i].elapsed_time(evs[i + 1]), 1), **host[i]})
    print(json.dumps({"args": vars(args), "plan": lms.plan_note, "plan_info": ctx.plan_info(), "steps": out},
                     indent=1))
    items = ctx.plan_items()
    if items:
        tag = "e2e" if args.e2e else "dev"
        with open(os.path.join(ROOT, "gpurun_out", f"b2b_items_{tag}.json"), "w") as fh:
            json.dump({"items": items, "limit": ctx.stats()["device_limit"]}, fh)


if __name__ == "__main__":
    main()
