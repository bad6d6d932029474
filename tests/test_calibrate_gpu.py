"""The calibrated model's measurements on the GPU (calibrate.node_costs,
LMS.plan_by_model): every captured forward/backward node gets a CUDA-event
time, the per-node times add up to the step's, and a ranking comes back for
candidate windows."""

import pytest
import torch

from paper_1807_02037_b200 import RewriteConfig
from paper_1807_02037_b200.calibrate import node_costs
from paper_1807_02037_b200.torch_lms import LMS

pytestmark = pytest.mark.gpu


def _net():
    torch.manual_seed(0)
    return torch.nn.Sequential(
        torch.nn.Conv2d(3, 32, 3, padding=1), torch.nn.BatchNorm2d(32), torch.nn.ReLU(inplace=True),
        torch.nn.Conv2d(32, 64, 3, padding=1), torch.nn.ReLU(),
        torch.nn.AdaptiveAvgPool2d(1), torch.nn.Flatten(), torch.nn.Linear(64, 10)).cuda()


def test_node_costs_cover_the_step(lms_ctx):
    net = _net()
    opt = torch.optim.SGD(net.parameters(), lr=0.1)
    lf = torch.nn.functional.cross_entropy
    lms = LMS(net, lf, opt, RewriteConfig(), lms_ctx, min_swap_bytes=0)
    x = torch.randn(32, 3, 64, 64, device="cuda")
    y = torch.randint(0, 10, (32,), device="cuda")
    lms.capture(x[:4], y[:4])
    costs = node_costs(net, lf, x, y, lms.meta, opt)
    f_ids, b_ids = set(lms.meta["F"]), set(lms.meta["B"])
    assert sum(1 for n in f_ids if costs.get(n, 0) > 0) >= len(f_ids) // 2
    assert sum(1 for n in b_ids if costs.get(n, 0) > 0) >= len(b_ids) // 2
    fwd = sum(costs.get(n, 0.0) for n in f_ids)
    assert fwd == pytest.approx(costs["_forward_total"], rel=0.25)
    assert sum(costs.get(n, 0.0) for n in b_ids) <= costs["_backward_total"] * 1.05
    link = lms.link_model({"d2h": 55.0, "h2d": 55.0})
    ranked = lms.plan_by_model(x, y, [RewriteConfig(lb=lb) for lb in (1, 2, 4)], 64, link, 8 << 30)
    assert len(ranked) == 3 and all(p["makespan"] > 0 for _, p, _ in ranked)
    assert ranked[0][2]
