"""Capture adapter (PyTorch autograd step -> CompGraph) on CPU.

The captured graph must be valid under the reference's ``validate`` rules,
carry forward/backward/update phases, and the reference rewrite must find the
saved activations as forward->backward candidates.
"""

import torch

from paper_1807_02037_b200 import EdgeAction, NodeKind, Phase, RewriteConfig, validate
from paper_1807_02037_b200.torch_lms import build_plan, capture_graph


def _model():
    torch.manual_seed(0)
    return torch.nn.Sequential(
        torch.nn.Conv2d(3, 8, 3, padding=1), torch.nn.BatchNorm2d(8), torch.nn.ReLU(),
        torch.nn.MaxPool2d(2),
        torch.nn.Conv2d(8, 16, 3, padding=1), torch.nn.ReLU(),
        torch.nn.Flatten(), torch.nn.Linear(16 * 8 * 8, 10))


def test_capture_is_valid_training_graph():
    m = _model()
    x = torch.randn(4, 3, 16, 16)
    y = torch.randint(0, 10, (4,))
    g, meta = capture_graph(lambda: torch.nn.functional.cross_entropy(m(x), y), min_swap_bytes=0)
    assert validate(g) == []
    phases = {n.phase for n in g.nodes if not n.parameterized}
    assert phases == {Phase.FORWARD, Phase.BACKWARD, Phase.UPDATE}
    n_params = sum(1 for _ in m.parameters())
    assert sum(1 for n in g.nodes if n.kind is NodeKind.VARIABLE) == n_params + 2
    fwd_bwd = [e for e in g.edges if e.action is EdgeAction.READ
               and g.node(e.src).phase is Phase.FORWARD and g.node(e.dst).phase is Phase.BACKWARD]
    assert len(fwd_bwd) >= 6  # conv inputs, bn input, relu outputs, pool indices, ...
    plan = build_plan(g, meta, RewriteConfig(), capture_batch=4)
    assert plan.report.tensors_swapped == len({e.tensor for e in fwd_bwd})
    assert len(plan.groups) == plan.report.swap_ins_added
    # every swapped pack is served by exactly one swap-in group
    served = sorted(k for grp in plan.groups for k in grp.packs)
    assert served == sorted(set(served))
    assert all(plan.pack_saved[k] >= 0 for k in served)
    kinds = {grp.trigger_kind for grp in plan.groups}
    assert "backward" in kinds


def test_n_tensors_and_fusion_knobs_apply():
    m = _model()
    x = torch.randn(2, 3, 16, 16)
    y = torch.randint(0, 10, (2,))
    g, meta = capture_graph(lambda: torch.nn.functional.cross_entropy(m(x), y), min_swap_bytes=0)
    p3 = build_plan(g, meta, RewriteConfig(n_tensors=3), capture_batch=2)
    assert p3.report.tensors_swapped == 3
    pf = build_plan(g, meta, RewriteConfig(fuse_swapins=True, swapin_fuse_distance=100), capture_batch=2)
    pn = build_plan(g, meta, RewriteConfig(), capture_batch=2)
    assert len(pf.groups) <= len(pn.groups)
    pd = build_plan(g, meta, RewriteConfig(ctrld_strategy="direct_order", lb=2), capture_batch=2)
    assert pd.report.control_edges_added > 0


def test_far_window_only_moves_small_tensors_triggers():
    """build_plan(far_cfg=...): same swap-ins as the plain rewrite; tensors under the
    size fraction take the far rewrite's control op, the rest keep their own."""
    import pytest
    m = _model()
    x = torch.randn(4, 3, 16, 16)
    y = torch.randint(0, 10, (4,))
    g, meta = capture_graph(lambda: torch.nn.functional.cross_entropy(m(x), y), min_swap_bytes=0)
    near = build_plan(g, meta, RewriteConfig(lb=1), 4)
    far = build_plan(g, meta, RewriteConfig(lb=3), 4)
    mixed = build_plan(g, meta, RewriteConfig(lb=1), 4, RewriteConfig(lb=3), 0.5)
    assert [grp.packs for grp in mixed.groups] == [grp.packs for grp in near.groups]
    biggest = max(s.nbytes for s in near.saved if s.swapped)
    for a, b, c in zip(near.groups, far.groups, mixed.groups):
        small = near.saved[a.saved].nbytes < 0.5 * biggest
        assert (c.trigger, c.trigger_kind) == ((b.trigger, b.trigger_kind) if small else (a.trigger, a.trigger_kind))
    with pytest.raises(ValueError):   # a far rewrite with other swap-ins is refused
        build_plan(g, meta, RewriteConfig(lb=1), 4, RewriteConfig(lb=3, n_tensors=1), 0.5)


def test_resnet50_capture_counts():
    """ResNet-50 (the headline model): every saved activation that outlives its
    forward op becomes a swap candidate; the rewrite is deterministic."""
    import torchvision
    torch.manual_seed(0)
    m = torchvision.models.resnet50()
    x = torch.randn(2, 3, 64, 64)
    y = torch.randint(0, 1000, (2,))
    persistent = list(m.parameters()) + list(m.buffers()) + [x, y]
    g, meta = capture_graph(lambda: torch.nn.functional.cross_entropy(m(x), y), 0, persistent)
    assert validate(g) == []
    a = build_plan(g, meta, RewriteConfig(fuse_swapins=True), 2)
    b = build_plan(g, meta, RewriteConfig(fuse_swapins=True), 2)
    assert a.report.to_dict() == b.report.to_dict()
    assert a.report.tensors_swapped >= 100          # conv/BN/ReLU activations of 53 convs
    assert len(a.groups) >= a.report.tensors_swapped
    assert not a.bwd_start_groups                   # chain_rule finds backward control ops
    capped = build_plan(g, meta, RewriteConfig(fuse_swapins=True, n_tensors=10), 2)
    assert capped.report.tensors_swapped == 10


def test_retarget_moves_triggers_and_keeps_issue_order():
    """retarget(plan, moves): the moved swap-ins fire from the new node, after that
    node's own swap-ins; every other group and the packs they serve are unchanged."""
    from paper_1807_02037_b200.torch_lms import retarget
    m = _model()
    x = torch.randn(4, 3, 16, 16)
    y = torch.randint(0, 10, (4,))
    g, meta = capture_graph(lambda: torch.nn.functional.cross_entropy(m(x), y), min_swap_bytes=0)
    near = build_plan(g, meta, RewriteConfig(lb=1), 4)
    far = build_plan(g, meta, RewriteConfig(lb=3), 4)
    assert [grp.node for grp in near.groups] == [grp.node for grp in far.groups]
    moves = {a.gid: b.trigger for a, b in zip(near.groups, far.groups)
             if a.trigger_kind == b.trigger_kind == "backward" and a.trigger != b.trigger}
    assert moves, "lb=3 should move at least one control op on this model"
    out = retarget(near, moves)
    for a, c in zip(near.groups, out.groups):
        assert c.packs == a.packs and c.node == a.node
        assert c.trigger == moves.get(a.gid, a.trigger)
    flat = sorted(gid for gids in out.triggers.values() for gid in gids)
    assert flat == sorted(gid for gids in near.triggers.values() for gid in gids)
    for r, gids in out.triggers.items():
        own = [gid for gid in near.triggers.get(r, []) if gid not in moves]
        assert gids[:len(own)] == own
    assert retarget(near, {}).triggers == near.triggers


def test_plan_window_moves_respects_room_and_issue_order():
    """The tune_windows model: each swap-in takes its earliest candidate whose
    window keeps live + bytes under the limit, never before the previous
    swap-in's trigger; accepted moves raise the live curve for later ones."""
    import numpy as np
    from paper_1807_02037_b200.torch_lms import plan_window_moves
    live = np.full(100, 10.0)
    live[20:30] = 18.0                      # a peak the first swap-in cannot span
    node_clock = {1: 10, 2: 35, 3: 40, 4: 50, 5: 60, 6: 5}
    issue = [(45, 0, 5.0), (70, 1, 4.0), (80, 2, 1.0)]
    cands = {0: [1, 2], 1: [3, 6], 2: [4, 5]}
    trig = {0: 9, 1: 9, 2: 5}
    out = plan_window_moves(live, node_clock, issue, cands, trig, limit=20.0)
    # gid 0: rank 1 (clock 10) spans the 18-byte peak (18 + 5 > 20) -> rank 2 (35)
    # gid 1: rank 6 (clock 5) would pass gid 0's new trigger -> rank 3 (40)
    # gid 2: rank 5 is its own trigger; rank 4 (50): live there is 10 + 4 + 1 <= 20
    assert [(g, c2, r) for g, _, c2, _, r in out] == [(0, 35, 2), (1, 40, 3), (2, 50, 4)]
    assert live[35:45].max() == 10 + 5 + 4 and live[60:70].max() == 10 + 4 + 1
    # no room at all: nothing moves
    live2 = np.full(100, 20.0)
    assert plan_window_moves(live2, node_clock, issue, cands, trig, limit=20.0) == []


def test_swap_branches_plans_forward_swaps():
    """swap_branches (rewriter.py:231) swaps fwd->fwd edges such as U-Net skip
    tensors; the plan maps them to forward-side swap-in groups (the round-1
    build_plan raised KeyError on them)."""
    from paper_1807_02037_b200.workloads import unet3d
    torch.manual_seed(0)
    m = unet3d(base=4, depth=2)
    x = torch.randn(1, 1, 16, 16, 16)
    y = torch.randint(0, 2, (1, 16, 16, 16))
    g, meta = capture_graph(lambda: torch.nn.functional.cross_entropy(m(x), y), min_swap_bytes=0)
    assert validate(g) == []
    assert meta["fwd_ranks_ok"]
    # forward outputs carry their bytes, so branch tensors have real sizes
    fwd_fwd = [e for e in g.edges if e.action is EdgeAction.READ and g.node(e.src).phase is Phase.FORWARD
               and g.node(e.dst).phase is Phase.FORWARD and g.tensor(e.tensor).size_bytes > 0]
    assert len(fwd_fwd) > 10
    plain = build_plan(g, meta, RewriteConfig(ctrld_strategy="chain_rule"), capture_batch=1)
    assert plain.fwd_groups == []
    cfg = RewriteConfig(swap_branches=True, branch_threshold=20, lb=1)
    plan = build_plan(g, meta, cfg, capture_batch=1)
    assert plan.report.swap_ins_added > plain.report.swap_ins_added
    fg = [plan.groups[i] for i in plan.fwd_groups]
    assert fg, "the skip concatenations' inputs are branch swaps"
    order = {}
    from paper_1807_02037_b200 import topo_order
    order = topo_order(g)
    for grp in fg:
        assert grp.fwd_consumers and grp.release_rank >= grp.producer_rank
        assert all(c > grp.release_rank for c in grp.fwd_consumers)
        if grp.trigger_kind == "forward":
            assert grp.release_rank <= grp.trigger < min(grp.fwd_consumers) or grp.trigger < grp.release_rank
        # the swapped edge jumps more than branch_threshold levels (strict >)
        t = g.tensor(grp.tensor)
        cons = [e.dst for e in g.consumer_edges(grp.tensor) if meta["F"].get(e.dst) in grp.fwd_consumers]
        assert all(order[d] - order[t.producer] > 20 for d in cons)
    # every group id indexes plan.groups
    assert [grp.gid for grp in plan.groups] == list(range(len(plan.groups)))
