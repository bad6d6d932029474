"""The calibrated step-time model (calibrate.py) on CPU: its list schedule agrees
with the reference model's serial peaks and makespans on plain graphs, transfers
stretch it only when the link is the bottleneck, and windows trade peak for time
(PAPER.md:951-963)."""

import math

import pytest

from paper_1807_02037_b200 import RewriteConfig, chain, rewrite, topo_order, unet
from paper_1807_02037_b200.calibrate import LinkModel, calibrated_graph, plan_ranking, predict
from oracle.sim_oracle import simulate as model

INF = LinkModel(math.inf, math.inf, math.inf, math.inf)


@pytest.mark.parametrize("g", [chain(20), unet(4, tensor_bytes=8 << 20)])
def test_plain_graph_matches_reference_serial_model(g):
    p = predict(g, INF)
    want = model(g, topo_order(g), serial=True, h2d_bw=math.inf, d2h_bw=math.inf)
    assert p["peak_device_bytes"] == want["peak_device_bytes"]
    assert p["makespan"] == pytest.approx(want["makespan"])
    assert p["d2h_busy"] == 0.0


def test_swaps_cost_nothing_on_an_infinite_link_and_time_on_a_slow_one():
    g = chain(20)
    g2, _ = rewrite(g, RewriteConfig())
    assert predict(g2, INF)["makespan"] == pytest.approx(predict(g, INF)["makespan"])
    slow = LinkModel(2**20, 2**20, 2**20, 2**20)      # 1 MiB/s: each 1 MiB tensor takes 1 s
    p = predict(g2, slow)
    assert p["d2h_busy"] == pytest.approx(20.0) and p["h2d_busy"] == pytest.approx(20.0)
    assert p["makespan"] > predict(g, INF)["makespan"]
    assert p["peak_device_bytes"] < predict(g, INF)["peak_device_bytes"]
    shared = LinkModel(2**20, 2**20, 2**20, 2**20, overlap=False)
    assert predict(g2, shared)["makespan"] >= p["makespan"]


def test_wider_windows_trade_memory_for_time():
    base = chain(30)
    g = calibrated_graph(base, {n.id: 0.5 for n in base.nodes}, 1.0)   # 0.5 s ops, 1 s transfers
    link = LinkModel(2**20, 2**20, 2**20, 2**20)
    cfgs = [RewriteConfig(lb=lb, ctrld_strategy="direct_order") for lb in (1, 2, 8, 16)]
    preds = {c.lb: p for c, p, _ in plan_ranking(g, cfgs, link, 1e18)}
    assert preds[8]["makespan"] < preds[2]["makespan"] < preds[1]["makespan"]
    assert preds[16]["peak_device_bytes"] > preds[1]["peak_device_bytes"]
    # a tight room: allocations wait for swap-out copies (the pool's throttle), the
    # peak stays under the room, and a room below one op's working set does not fit
    tight = {c.lb: (p, fit) for c, p, fit in plan_ranking(g, cfgs, link, 4 << 20)}
    for lb, (p, fit) in tight.items():
        assert fit and p["peak_device_bytes"] <= 4 << 20 and p["alloc_stall"] > 0
        assert p["makespan"] >= preds[lb]["makespan"]
    assert not any(fit for _, _, fit in plan_ranking(g, cfgs, link, 1 << 20))


def test_wire_ratio_shortens_transfers():
    g2, _ = rewrite(chain(10), RewriteConfig())
    swapped = {t.id for t in chain(10).tensors}
    full = predict(g2, LinkModel(2**20, 2**20, 2**20, 2**20))
    half = predict(g2, LinkModel(2**20, 2**20, 2**20, 2**20, wire_ratio={t: 0.5 for t in swapped}))
    assert half["d2h_busy"] == pytest.approx(full["d2h_busy"] / 2)
