"""Where does a swapped ResNet step spend its time?  Forward/backward windows vs link busy time.

Usage: python scripts/step_timeline.py --batch 908 [--budget-gib 16] [--codec auto] [--lb 1] [--n-tensors -1]
Prints per-window: duration, D2H / H2D busy (union of transfer spans), link-idle time, and
the largest gaps between consecutive transfers with the compute op near each gap.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def union(spans, lo, hi):
    spans = sorted((max(a, lo), min(b, hi)) for a, b in spans if b > lo and a < hi)
    tot, cur_a, cur_b = 0.0, None, None
    for a, b in spans:
        if cur_b is None or a > cur_b:
            if cur_b is not None:
                tot += cur_b - cur_a
            cur_a, cur_b = a, b
        else:
            cur_b = max(cur_b, b)
    if cur_b is not None:
        tot += cur_b - cur_a
    return tot


def gaps(spans, lo, hi, k=5):
    spans = sorted((a, b) for a, b in spans if b > lo and a < hi)
    out, t = [], lo
    for a, b in spans:
        if a > t:
            out.append((a - t, t, a))
        t = max(t, b)
    if hi > t:
        out.append((hi - t, t, hi))
    return sorted(out, reverse=True)[:k]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=908)
    ap.add_argument("--budget-gib", type=float, default=16.0)
    ap.add_argument("--codec", default="auto")
    ap.add_argument("--tf32", action="store_true")
    ap.add_argument("--lb", type=int, default=1)
    ap.add_argument("--ub", type=int, default=10000)
    ap.add_argument("--strategy", default="chain_rule")
    ap.add_argument("--n-tensors", type=int, default=-1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--no-plan", action="store_true")
    ap.add_argument("--fuse-distance", type=int, default=1)
    ap.add_argument("--tune", action="store_true", help="LMS.tune_windows before the traced steps")
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
    cfg = RewriteConfig(lb=args.lb, ub=args.ub, ctrld_strategy=args.strategy, fuse_swapins=True,
                        swapin_fuse_distance=args.fuse_distance, n_tensors=args.n_tensors)
    lms = LMS(model, lf, opt, cfg, ctx, codec=args.codec, min_swap_bytes=(256 << 10) // 4,
              static_plan=not args.no_plan)
    xc = torch.randn(4, 3, 224, 224, device=dev)
    yc = torch.randint(0, 1000, (4,), device=dev)
    lms.capture(xc, yc)
    del xc, yc
    x = torch.randn(args.batch, 3, 224, 224, device=dev)
    y = torch.randint(0, 1000, (args.batch,), device=dev)
    s = torch.cuda.current_stream()
    marks = {}
    tuned = lms.tune_windows(x, y) if args.tune else None

    run = lms._exec.run

    def run_marked(forward_fn):
        def fwd():
            out = forward_fn()
            marks["fwd_end"].record(s)
            return out
        return run(fwd)

    lms._exec.run = run_marked

    for step in range(args.steps):
        torch.cuda.synchronize()
        ctx.synchronize()
        ctx.trace_clear()
        ev = {k: torch.cuda.Event(enable_timing=True) for k in ("start", "fwd_end", "end")}
        marks.update(ev)
        # the epoch event lives on the D2H stream; make the start event comparable
        d2h, _ = ctx.streams()
        epoch = torch.cuda.Event(enable_timing=True)
        epoch.record(d2h)
        st0 = ctx.stats()
        ev["start"].record(s)
        lms.step(x, y)
        ev["end"].record(s)
        torch.cuda.synchronize()
        ctx.synchronize()
        tr = ctx.trace()
    # times in ms relative to the context epoch (trace_clear re-records it on the D2H stream)
    t0 = epoch.elapsed_time(ev["start"])
    tf = epoch.elapsed_time(ev["fwd_end"])
    te = epoch.elapsed_time(ev["end"])
    d2h = [(r["start_ms"], r["end_ms"]) for r in tr if r["direction"] == 0]
    h2d = [(r["start_ms"], r["end_ms"]) for r in tr if r["direction"] == 1]
    both = d2h + h2d
    st = ctx.stats()
    res = {
        "batch": args.batch, "codec": args.codec, "lb": args.lb, "plan": lms.plan.summary(), "tune_windows": tuned,
        "step_ms": te - t0, "fwd_ms": tf - t0, "bwd_opt_ms": te - tf,
        "fwd": {"d2h_busy": union(d2h, t0, tf), "h2d_busy": union(h2d, t0, tf), "any_busy": union(both, t0, tf)},
        "bwd": {"d2h_busy": union(d2h, tf, te), "h2d_busy": union(h2d, tf, te), "any_busy": union(both, tf, te)},
        "d2h_total_busy": union(d2h, -1e9, 1e9), "h2d_total_busy": union(h2d, -1e9, 1e9),
        "d2h_GB": sum(r["wire_bytes"] for r in tr if r["direction"] == 0) / 1e9,
        "h2d_GB": sum(r["wire_bytes"] for r in tr if r["direction"] == 1) / 1e9,
        "last_d2h_end": max((b for _, b in d2h), default=0) - t0,
        "first_h2d_start": min((a for a, _ in h2d), default=0) - t0,
        "fwd_gaps_d2h": [(round(g, 2), round(a - t0, 1)) for g, a, _ in gaps(d2h, t0, tf)],
        "bwd_gaps_h2d": [(round(g, 2), round(a - t0, 1)) for g, a, _ in gaps(h2d, tf, te)],
        "swap_wait_ms": st["swap_wait_ms"], "n_device_syncs": st["n_device_syncs"],
        "alloc_wait_ms": st["alloc_wait_ms"] - st0["alloc_wait_ms"], "host_grow_ms": st["host_grow_ms"] - st0["host_grow_ms"],
        "n_host_grow": st["n_host_grow"] - st0["n_host_grow"], "n_scratch_grow": st["n_scratch_grow"] - st0["n_scratch_grow"],
        "pool_driver_ms": st["pool_driver_ms"] - st0["pool_driver_ms"], "n_reclaims": st["n_reclaims"] - st0["n_reclaims"],
        "unmap_ms": st["unmap_ms"] - st0["unmap_ms"], "map_ms": st["map_ms"] - st0["map_ms"],
        "access_ms": st["access_ms"] - st0["access_ms"], "n_map": st["n_map"] - st0["n_map"],
        "device_peak_GB": st["device_peak"] / 1e9, "plan_info": ctx.plan_info(),
    }
    print(json.dumps(res, indent=1))
    # Chrome trace (chrome://tracing / Perfetto) of the last step: compute windows and
    # every transfer on its copy channel, from CUDA events (no nsys in this image)
    ev = [{"name": "forward", "ph": "X", "pid": 0, "tid": 0, "ts": 0.0, "dur": (tf - t0) * 1e3},
          {"name": "backward+optimizer", "ph": "X", "pid": 0, "tid": 0, "ts": (tf - t0) * 1e3,
           "dur": (te - tf) * 1e3}]
    names = {0: "copy-engine", 1: "sm-zero-copy", 2: "zvc", 3: "zx"}
    for r in tr:
        ev.append({"name": f"{'swap-out' if r['direction'] == 0 else 'swap-in'} {names.get(r['codec'])} "
                           f"{r['logical_bytes'] / 2**20:.0f} MiB -> {r['wire_bytes'] / 2**20:.0f} MiB",
                   "ph": "X", "pid": 0, "tid": 1 + r["direction"], "ts": (r["start_ms"] - t0) * 1e3,
                   "dur": (r["end_ms"] - r["start_ms"]) * 1e3})
    meta = [{"name": "thread_name", "ph": "M", "pid": 0, "tid": k, "args": {"name": n}}
            for k, n in ((0, "compute stream"), (1, "D2H channel"), (2, "H2D channel"))]
    with open(os.path.join(ROOT, "gpurun_out", f"timeline_{args.codec}_{args.batch}.json"), "w") as fh:
        json.dump({"traceEvents": meta + ev, "displayTimeUnit": "ms"}, fh)
    items = ctx.plan_items()
    if items:
        with open(os.path.join(ROOT, "gpurun_out", f"plan_items_{args.codec}_{args.batch}.json"), "w") as fh:
            json.dump({"items": items, "limit": st["device_limit"], "in_use_end": st["device_in_use"]}, fh)


if __name__ == "__main__":
    main()
