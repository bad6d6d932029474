"""The measured ``simulate`` (simulate.py) against the reference's model.

The reference's ``simulate(g, order, SimConfig)`` (sim.py:139-476) models
peaks and transfers; ours runs the same schedule on the B200 through liblms
(real pool blocks, real D2H/H2D copies, a verifying payload kernel per op).
Checked here:

* plain graphs: the measured device peak equals the model's exactly (sizes
  are pool-granule multiples; no transfers, so alloc/free order is the serial
  schedule's), against the oracle restatement pinned to the reference;
* rewritten graphs: every swap chain delivers the producer's bytes (the
  payload kernel verifies each input word), the schedule runs inside the
  plain run's peak as its budget, and the D2H/H2D traffic is exactly the
  swapped bytes;
* the budget: a capacity below the plain peak reports ``oom=True`` and still
  completes (sim.py:471); the rewritten graph under the capacity the model
  says it needs does not;
* ``overlap_transfers=False`` puts D2H and H2D on one channel: no two
  transfers overlap in time (sim.py:284-290).
"""

import pytest

from paper_1807_02037_b200 import (
    RewriteConfig,
    SimConfig,
    chain,
    free_step_oracle,
    rewrite,
    simulate,
    topo_order,
    unet,
)
from oracle.sim_oracle import simulate as model

pytestmark = pytest.mark.gpu
MIB = 1 << 20


def _graphs():
    yield "chain(20)", chain(20)
    yield "unet(4,8MiB)", unet(4, tensor_bytes=8 * MIB)


@pytest.mark.parametrize("name,g", list(_graphs()))
def test_plain_peak_equals_model(lms_ctx, name, g):
    order = topo_order(g)
    got = simulate(g, order, SimConfig.serial_oracle())
    want = model(g, order, serial=True, h2d_bw=float("inf"), d2h_bw=float("inf"))
    assert got.peak_device_bytes == want["peak_device_bytes"], name
    assert got.peak_host_bytes == 0 and not got.oom
    assert got.transfer_time_total == 0.0
    starts = [e for e in got.event_trace if e.event == "start"]
    assert len(starts) == sum(1 for n in g.nodes if not n.parameterized)


@pytest.mark.parametrize("cfg", [RewriteConfig(), RewriteConfig(lb=2, ctrld_strategy="direct_order"),
                                 RewriteConfig(lb=1, swap_branches=True, branch_threshold=1,
                                               ctrld_strategy="direct_order", fuse_swapins=True)])
def test_rewritten_schedule_moves_exact_bytes(lms_ctx, cfg):
    g = unet(4, tensor_bytes=8 * MIB)
    plain = simulate(g, topo_order(g), SimConfig())
    g2, rep = rewrite(g, cfg)
    order = topo_order(g2)
    # without a tight budget the compute stream runs ahead of the D2H channel and
    # swapped-out blocks stay held until their copies land, so the peak is only
    # bounded once the budget makes allocations wait for them (sim.py:205-211)
    cap = SimConfig(device_capacity_bytes=plain.peak_device_bytes)
    got = simulate(g2, order, cap)               # verify=True: wrong bytes raise
    assert not got.oom and got.peak_device_bytes <= plain.peak_device_bytes
    xs = [e for e in got.event_trace if e.event == "xfer_finish"]
    d2h = sum(e.bytes for e in xs if e.device == "host")
    h2d = sum(e.bytes for e in xs if e.device != "host")
    assert d2h == rep.swap_outs_added * 8 * MIB
    assert h2d == rep.swap_ins_added * 8 * MIB
    assert got.peak_host_bytes <= rep.swap_outs_added * 8 * MIB
    assert got.transfer_time_total > 0 and got.makespan > 0
    # every swapped tensor's free step in the rewritten schedule is the model's
    for t in g2.tensors:
        free_step_oracle(g2, order, t.id)


def test_budget_reports_oom_and_completes(lms_ctx):
    g = chain(20)
    order = topo_order(g)
    want = model(g, order, serial=True, h2d_bw=float("inf"), d2h_bw=float("inf"))["peak_device_bytes"]
    r = simulate(g, order, SimConfig(device_capacity_bytes=want // 2))
    assert r.oom and r.peak_device_bytes >= want
    r = simulate(g, order, SimConfig(device_capacity_bytes=want))
    assert not r.oom


def test_rewrite_fits_the_models_capacity(lms_ctx):
    # the reference acceptance case (test_acceptance.py:171-180): unet(4, 8 MiB),
    # lb=1 with branches, <= half the plain peak in the model.  The pool holds
    # swapped-out blocks until their copies land and allocations wait for them,
    # so the real schedule runs inside the plain peak without an OOM.
    g = unet(4, tensor_bytes=8 * MIB)
    cfg = RewriteConfig(lb=1, swap_branches=True, branch_threshold=1, ctrld_strategy="direct_order")
    g2, _ = rewrite(g, cfg)
    o2 = topo_order(g2)
    plain = model(g, topo_order(g))["peak_device_bytes"]
    swapped = model(g2, o2)["peak_device_bytes"]
    assert swapped <= plain // 2
    r = simulate(g2, o2, SimConfig(device_capacity_bytes=plain))
    assert not r.oom and r.peak_device_bytes <= plain


def test_shared_channel_serialises_transfers(lms_ctx):
    g = unet(4, tensor_bytes=8 * MIB)
    g2, _ = rewrite(g, RewriteConfig(lb=1, swap_branches=True, branch_threshold=1,
                                     ctrld_strategy="direct_order"))
    r = simulate(g2, topo_order(g2), SimConfig(overlap_transfers=False))
    spans = []
    open_at = {}
    for e in r.event_trace:
        if e.event == "xfer_start":
            open_at.setdefault((e.tensor, e.device), []).append(e.time)
        elif e.event == "xfer_finish":
            spans.append((open_at[(e.tensor, e.device)].pop(0), e.time, e.device))
    spans.sort()
    assert len(spans) >= 8
    eps = 2e-6   # CUDA event resolution
    for (a0, a1, _), (b0, b1, _) in zip(spans, spans[1:]):
        assert b0 >= a1 - eps, (a0, a1, b0, b1)
