"""The capture recipe behind captured_cases.json.gz (shared by make_captured.py
and tests/test_captured_parity.py; imports nothing from the reference)."""

from __future__ import annotations

MIN_SWAP = 64 << 10


def capture(name):
    """The captured graph of one workload (CPU, fixed seed)."""
    import torch
    import torchvision
    from paper_1807_02037_b200.torch_lms import capture_graph
    from paper_1807_02037_b200.workloads import unet3d
    torch.manual_seed(0)
    if name == "resnet50":
        m, x = torchvision.models.resnet50(), torch.randn(4, 3, 224, 224)
        y = torch.randint(0, 1000, (4,))
    elif name == "resnet152":
        m, x = torchvision.models.resnet152(), torch.randn(1, 3, 224, 224)
        y = torch.randint(0, 1000, (1,))
    else:
        m, x = unet3d(), torch.randn(1, 1, 32, 32, 32)
        y = torch.randint(0, 2, (1, 32, 32, 32))
    persistent = list(m.parameters()) + list(m.buffers()) + [x, y]
    g, _ = capture_graph(lambda: torch.nn.functional.cross_entropy(m(x), y), MIN_SWAP, persistent)
    return g
