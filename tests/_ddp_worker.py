"""Worker for tests/test_ddp_gpu.py: data-parallel training, one process per rank.

Launched as ``python -m torch.distributed.run --nproc-per-node 2 tests/_ddp_worker.py
MODE OUTDIR [BUDGET_GIB]`` with both ranks on cuda:0 (the gloo backend moves the
gradient all-reduce through the host, so two ranks can share one GPU).  Each
rank owns its liblms pool; MODE ``swap`` trains through TFLMS (capture ->
reference rewrite -> swap engine, static plan, tune_windows with its decisions
agreed across ranks), MODE ``plain`` trains without it.  Every rank writes its
losses and final state_dict to OUTDIR/MODE_rank{r}.pt.
"""

from __future__ import annotations

import copy
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GIB = 1 << 30


def main():
    mode, outdir = sys.argv[1], sys.argv[2]
    budget = float(sys.argv[3]) if len(sys.argv) > 3 else 8.0
    import torch
    import torch.distributed as dist
    import torchvision
    from paper_1807_02037_b200 import RewriteConfig, runtime as rt
    from paper_1807_02037_b200.torch_lms import LMS

    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ctx = rt.Context(device=0, device_reserve=int(budget * GIB), host_chunk=1 << 30, timing=True)
    rt.install_allocator(ctx)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    torch.manual_seed(0)
    base = torchvision.models.resnet18().cuda()
    init = copy.deepcopy(base.state_dict())
    model = torch.nn.parallel.DistributedDataParallel(base, device_ids=[0])
    opt = torch.optim.SGD(model.parameters(), lr=0.01, momentum=0.9)
    loss_fn = torch.nn.functional.cross_entropy

    def batch(i, n=64):
        g = torch.Generator(device="cuda").manual_seed(100 * i + rank)   # each rank its own shard
        return (torch.randn(n, 3, 160, 160, device="cuda", generator=g),
                torch.randint(0, 1000, (n,), device="cuda", generator=g))

    def agree(v, op):
        t = torch.tensor([float(v)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.MIN)
        return t.item()

    steps = 4
    batches = [batch(i) for i in range(steps)]
    facts = {}
    if mode == "plain":
        losses = []
        for x, y in batches:
            opt.zero_grad(set_to_none=True)
            loss = loss_fn(model(x), y)
            loss.backward()
            opt.step()
            losses.append(loss.detach().clone())
        facts["peak"] = ctx.stats()["device_peak"]
    else:
        lms = LMS(model, loss_fn, opt, RewriteConfig(lb=1, fuse_swapins=True, swapin_fuse_distance=12), ctx,
                  codec="auto")
        lms.capture(*batch(99, 4))
        facts["tuned"] = lms.tune_windows(*batches[0], steps=2, agree=agree)
        # under DDP the tuner runs the local replica and restores the training state
        facts["tune_restored"] = all(torch.equal(v, init[k]) for k, v in base.state_dict().items())
        ctx.trace_clear()
        losses = [lms.step(x, y).detach().clone() for x, y in batches]
        torch.cuda.synchronize()
        st = ctx.stats()
        facts.update(peak=st["device_peak"], d2h=st["d2h_logical_bytes"], plan_note=lms.plan_note,
                     swapped=lms.plan.report.tensors_swapped)
    torch.save({"losses": [l.cpu() for l in losses],
                "state": {k: v.detach().cpu() for k, v in base.state_dict().items()}, "facts": facts},
               os.path.join(outdir, f"{mode}_rank{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}/{ws} {mode} ok {facts}")


if __name__ == "__main__":
    main()
