"""Worker for tests/test_model_parity_gpu.py: one training run in its own process.

Each run owns a fresh liblms pool sized like the bench's (the pool's physical
pages ARE the budget, so the static plan places exactly as in `bench.py`):

    python tests/_parity_worker.py plain  MODEL OUT.pt [--budget-gib G]
    python tests/_parity_worker.py swap   MODEL OUT.pt --budget-gib G [--tune] [--branches]

MODEL is ``resnet50`` (batch 96, 224^2) or ``unet3d`` (batch 2, 64^3).  Writes
the per-step losses, the final state_dict and run facts to OUT.pt.
"""

from __future__ import annotations

import argparse
import copy
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GIB = 1 << 30


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["plain", "swap"])
    ap.add_argument("model", choices=["resnet50", "unet3d"])
    ap.add_argument("out")
    ap.add_argument("--budget-gib", type=float, default=40.0)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--tune", action="store_true")
    ap.add_argument("--branches", action="store_true")
    ap.add_argument("--page-mb", type=int, default=0, help="pool page size (small budgets want small pages)")
    a = ap.parse_args()
    if a.page_mb:
        os.environ["LMS_PAGE_MB"] = str(a.page_mb)

    import torch
    from paper_1807_02037_b200 import RewriteConfig, runtime as rt
    from paper_1807_02037_b200.torch_lms import LMS

    budget = int(a.budget_gib * GIB)
    ctx = rt.Context(device=0, device_reserve=budget, host_chunk=2 * GIB, timing=True)
    rt.install_allocator(ctx)
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    torch.manual_seed(0)
    if a.model == "resnet50":
        import torchvision
        model = torchvision.models.resnet50().cuda()
        B, cap_b = 96, 4

        def batch(i, n=B):
            g = torch.Generator(device="cuda").manual_seed(1000 + i)
            return (torch.randn(n, 3, 224, 224, device="cuda", generator=g),
                    torch.randint(0, 1000, (n,), device="cuda", generator=g))
        cfg = RewriteConfig(lb=1, ctrld_strategy="chain_rule", fuse_swapins=True, swapin_fuse_distance=12)
    else:
        from paper_1807_02037_b200.workloads import unet3d
        model = unet3d().cuda()
        B, cap_b = 2, 1

        def batch(i, n=B):
            g = torch.Generator(device="cuda").manual_seed(2000 + i)
            s = 32 if i == 99 else 64
            return (torch.randn(n, 1, s, s, s, device="cuda", generator=g),
                    torch.randint(0, 2, (n, s, s, s), device="cuda", generator=g))
        cfg = RewriteConfig(lb=1, ctrld_strategy="chain_rule", swap_branches=a.branches, branch_threshold=20)
    init = copy.deepcopy(model.state_dict())
    loss_fn = torch.nn.functional.cross_entropy
    opt = torch.optim.SGD(model.parameters(), lr=0.01, momentum=0.9)
    batches = [batch(i) for i in range(a.steps)]
    facts = {"budget": budget}
    torch.cuda.synchronize()
    if a.mode == "plain":
        ctx.reset_peaks()
        base = ctx.stats()["device_in_use"]
        losses = []
        for x, y in batches:
            opt.zero_grad(set_to_none=True)
            loss = loss_fn(model(x), y)
            loss.backward()
            opt.step()
            losses.append(loss.detach().clone())
        torch.cuda.synchronize()
        facts["peak"] = ctx.stats()["device_peak"]
        facts["peak_over_base"] = facts["peak"] - base
    else:
        lms = LMS(model, loss_fn, opt, cfg, ctx, codec="auto")
        lms.capture(*batch(99, cap_b))
        if a.tune:
            facts["tuned"] = lms.tune_windows(*batches[0])
            model.load_state_dict(init)            # the tuner's trial steps moved the weights
            opt.state.clear()
        torch.cuda.synchronize()
        ctx.trace_clear()
        ctx.reset_peaks()
        losses = [lms.step(x, y).detach().clone() for x, y in batches]
        torch.cuda.synchronize()
        st = ctx.stats()
        fwd = lms._exec.forward_swaps
        facts.update(peak=st["device_peak"], d2h=st["d2h_logical_bytes"], h2d=st["h2d_logical_bytes"],
                     n_oom=st["n_oom"],
                     plan_note=lms.plan_note, plan=ctx.plan_info(), summary=lms.plan.summary(),
                     forward_freed=fwd.n_freed if fwd is not None else 0)
    torch.save({"losses": [l.cpu() for l in losses],
                "state": {k: v.detach().cpu() for k, v in model.state_dict().items()},
                "facts": facts}, a.out)
    print("worker ok", {k: v for k, v in facts.items() if k not in ("plan", "summary")})


if __name__ == "__main__":
    main()
