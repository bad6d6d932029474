"""Data-parallel replicas on CPU: world_size 2 over gloo.

Each rank captures its DDP-wrapped training step and rewrites it.  The swap
schedule must be identical on every rank (same graph, same rewrite bytes),
since the replicas swap independently but must stay in lock-step around
the gradient allreduce, and the allreduced gradients must agree.
"""

import hashlib
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _net():
    torch.manual_seed(0)
    return torch.nn.Sequential(
        torch.nn.Conv2d(3, 16, 3, padding=1), torch.nn.BatchNorm2d(16), torch.nn.ReLU(inplace=True),
        torch.nn.MaxPool2d(2),
        torch.nn.Conv2d(16, 32, 3, padding=1), torch.nn.ReLU(),
        torch.nn.AdaptiveAvgPool2d(1), torch.nn.Flatten(), torch.nn.Linear(32, 10))


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1807_02037_b200 import RewriteConfig, dumps
        from paper_1807_02037_b200.torch_lms import build_plan, capture_graph

        model = torch.nn.parallel.DistributedDataParallel(_net())
        g = torch.Generator().manual_seed(100 + rank)   # each replica its own shard
        x = torch.randn(8, 3, 16, 16, generator=g)
        y = torch.randint(0, 10, (8,), generator=g)
        persistent = list(model.parameters()) + list(model.buffers()) + [x, y]
        graph, meta = capture_graph(lambda: torch.nn.functional.cross_entropy(model(x), y), 0, persistent)
        plan = build_plan(graph, meta, RewriteConfig(lb=1, fuse_swapins=True), 8)
        digest = hashlib.sha256(dumps(plan.rewritten).encode()).hexdigest()
        grads = torch.cat([p.grad.flatten() for p in model.parameters()])
        gathered = [None] * world
        dist.all_gather_object(gathered, {"digest": digest, "summary": plan.summary(),
                                          "grads": grads.tolist()})
        if rank == 0:
            out.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_replicas_rewrite_identically_and_allreduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = res
    assert a["digest"] == b["digest"]
    sa = dict(a["summary"])
    sb = dict(b["summary"])
    sa.pop("rewrite_seconds")
    sb.pop("rewrite_seconds")
    assert sa == sb and sa["tensors_swapped"] > 0
    ga, gb = torch.tensor(a["grads"]), torch.tensor(b["grads"])
    assert torch.allclose(ga, gb, rtol=0, atol=0)   # DDP averaged the same bytes on both ranks
