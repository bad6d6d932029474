"""CPU baseline of the executor path for model-scale configs — TEST/BENCH INFRASTRUCTURE.

The reference executor (``interp.py:58-163``) runs the rewritten graph
serially on the host with swap nodes as identities that move no bytes
(``interp.py:168-170``), and its op vocabulary cannot express convolutions.
For the ResNet configs the CPU restatement of that executor is therefore:
the same training step (forward, backward, SGD momentum update) on the host
cores in fp32, with every swap an identity — i.e. a plain CPU step, which is
exactly what the reference's semantics reduce to.  Only ``bench.py`` (its
cpu_baseline leg and ``--impl reference``) and tests may use this module.
"""

from __future__ import annotations

import os
import time


def resnet_cpu_step_rate(arch: str = "resnet50", batch: int = 8, steps: int = 3, warmup: int = 1,
                         threads: int | None = None, image: int = 224, budget_s: float = 30.0):
    """img/s of fp32 training steps on the host; returns (img_per_s, threads, detail)."""
    import torch
    import torchvision

    threads = threads or len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    torch.manual_seed(0)
    if arch == "unet3d":
        from paper_1807_02037_b200.workloads import unet3d   # the model definition only
        model = unet3d()
        x = torch.randn(batch, 1, image, image, image)
        y = torch.randint(0, 2, (batch, image, image, image))
    else:
        model = getattr(torchvision.models, arch)()
        x = torch.randn(batch, 3, image, image)
        y = torch.randint(0, 1000, (batch,))
    model.train()
    opt = torch.optim.SGD(model.parameters(), lr=0.1, momentum=0.9)

    def step():
        opt.zero_grad(set_to_none=True)
        loss = torch.nn.functional.cross_entropy(model(x), y)
        loss.backward()
        opt.step()
        return loss

    for _ in range(warmup):
        step()
    t0 = time.perf_counter()
    done = 0
    while done < steps:
        step()
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return batch * done / dt, threads, {"batch": batch, "steps": done, "seconds": dt, "arch": arch}
