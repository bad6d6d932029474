"""Calibrated step-time model: pick lb / n_tensors by prediction.

The paper leaves choosing the swap window and the number of swapped tensors to
the user; the reference's simulator models a step from
``cost_hint`` and link bandwidths (sim.py:139-476) but nothing sets those from
a real run.  Here they come from measurements on the B200:

* ``node_costs`` times one plain step per autograd node with CUDA events —
  forward ops from a TorchFunctionMode that records an event after each op
  (the node's rank identifies its F node), backward nodes from pre/post hooks
  on every autograd node, the optimizer step as one span split over the
  update nodes;
* ``calibrated_graph`` writes those seconds into the captured graph's
  ``cost_hint`` and scales its tensor sizes to the target batch;
* ``LinkModel`` holds the copy-engine and zero-copy rates of each direction
  and each swapped tensor's wire ratio (the capture step's ZX estimate);
* ``predict`` runs a rewritten graph through a list-scheduling model of the
  executor: ops in the serial (order, id) sequence on one compute stream,
  swap-outs and swap-ins in issue order on their copy channels (one shared
  channel without overlap), each swap-in gated by its control op and its
  swap-out — the same gating the GPU executor uses — with allocations
  throttled by the room the budget leaves (an op waits for already-known
  frees, as the pool makes it wait for swap-out copies); it reports the
  makespan, the link busy time, the allocation stalls, the activation peak
  and whether the step fits (tensors allocated at their producer's start,
  released after their last reader, a swapped tensor only after its copy
  landed: sim.py:205-211);
* ``LMS.plan_by_model`` ranks candidate ``RewriteConfig``s by predicted step
  time among those whose predicted peak fits the budget.

The model is a predictor, not a test oracle: the chosen configuration is
then timed for real (``bench.py --model-select``), and the prediction error
is reported next to it.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import torch

from .graph import CompGraph, EdgeAction, NodeKind, TensorSpec, topo_order
from .simulate import _exec_set, _schedule


def node_costs(model, loss_fn, x, y, meta: dict, optimizer=None) -> dict[int, float]:
    """Seconds per captured node (F, B and update nodes) from one plain step at (x, y).

    ``meta`` is the capture's (``LMS.meta``): its F/B maps give node id ->
    autograd rank.  The step runs without swapping (x, y must fit)."""
    from torch.overrides import TorchFunctionMode
    from torch.utils._pytree import tree_flatten

    s = torch.cuda.current_stream()
    fwd_marks: list[tuple[int, torch.cuda.Event]] = []
    seq0 = [None]

    class _Marks(TorchFunctionMode):
        def __torch_function__(self, func, types, args=(), kwargs=None):
            out = func(*args, **(kwargs or {}))
            ranks = set()
            for t in tree_flatten(out)[0]:
                if isinstance(t, torch.Tensor) and t.grad_fn is not None:
                    seq = t.grad_fn._sequence_nr()
                    if seq0[0] is None:
                        seq0[0] = seq
                    ranks.add(seq - seq0[0])
            if ranks:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(s)
                fwd_marks.append((max(ranks), ev))
            return out

    if optimizer is not None:
        optimizer.zero_grad(set_to_none=True)
    start = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(s)
    with _Marks():
        loss = loss_fn(model(x), y)
    fwd_end = torch.cuda.Event(enable_timing=True)
    fwd_end.record(s)
    # backward: a pre- and a post-hook on every autograd node
    nodes, todo, seen = [], [loss.grad_fn], set()
    while todo:
        n = todo.pop()
        if n is None or n in seen:
            continue
        seen.add(n)
        nodes.append(n)
        todo.extend(nx for nx, _ in n.next_functions)
    bw_ev: dict = {}
    hooks = []
    for n in nodes:
        if n.name() == "torch::autograd::AccumulateGrad":
            continue

        def pre(grad_out, n=n):
            e = torch.cuda.Event(enable_timing=True)
            e.record(torch.cuda.current_stream())
            bw_ev.setdefault(n, [None, None])[0] = e

        def post(grad_in, grad_out, n=n):
            e = torch.cuda.Event(enable_timing=True)
            e.record(torch.cuda.current_stream())
            bw_ev.setdefault(n, [None, None])[1] = e

        hooks.append(n.register_prehook(pre))
        hooks.append(n.register_hook(post))
    try:
        loss.backward()
    finally:
        for h in hooks:
            h.remove()
    opt_a = torch.cuda.Event(enable_timing=True)
    opt_a.record(s)
    if optimizer is not None:
        optimizer.step()
    opt_b = torch.cuda.Event(enable_timing=True)
    opt_b.record(s)
    torch.cuda.synchronize()
    if optimizer is not None:
        optimizer.zero_grad(set_to_none=True)

    costs: dict[int, float] = {}
    F, B = meta["F"], meta["B"]          # node id -> rank
    f_of = {r: nid for nid, r in F.items()}
    b_of = {r: nid for nid, r in B.items()}
    # forward: each mark closes the ops since the previous one; charge it to its node
    prev = start
    for r, ev in fwd_marks:
        dt = prev.elapsed_time(ev) * 1e-3
        if r in f_of:
            costs[f_of[r]] = costs.get(f_of[r], 0.0) + max(dt, 0.0)
        prev = ev
    seqs = sorted(n._sequence_nr() for n in nodes if n.name() != "torch::autograd::AccumulateGrad")
    base = seqs[0] if seqs else 0
    for n, (a, b) in bw_ev.items():
        r = n._sequence_nr() - base
        if a is not None and b is not None and r in b_of:
            costs[b_of[r]] = max(a.elapsed_time(b) * 1e-3, 0.0)
    costs["_forward_total"] = start.elapsed_time(fwd_end) * 1e-3
    costs["_backward_total"] = fwd_end.elapsed_time(opt_a) * 1e-3
    costs["_optimizer_total"] = opt_a.elapsed_time(opt_b) * 1e-3
    return costs


def calibrated_graph(g: CompGraph, costs: dict, size_scale: float, cost_scale: float = 1.0,
                     update_total: float = 0.0, meta: dict | None = None) -> CompGraph:
    """``g`` with measured ``cost_hint`` seconds (x cost_scale) and tensor sizes x size_scale.

    With the capture's ``meta``, the backward ops' gradient tensors (sized 0 by
    the capture: autograd does not save them) get the size of the forward
    outputs they are the gradients of, so the model sees backward memory."""
    if meta is not None:
        F_of_rank = {r: nid for nid, r in meta["F"].items()}
        main_out = {}
        for t in g.tensors:
            if t.producer in meta["F"] and t.producer not in main_out:
                main_out[t.producer] = t.size_bytes     # the F node's first tensor: its output
        sized = []
        for t in g.tensors:
            if t.size_bytes == 0 and t.producer in meta["B"]:
                # consumers B(m): this tensor carries the gradient of m's forward output
                ranks = {meta["B"][e.dst] for e in g.consumer_edges(t.id) if e.dst in meta["B"]}
                nb = sum(main_out.get(F_of_rank.get(r), 0) for r in ranks)
                t = TensorSpec(t.id, t.producer, nb, t.dtype)
            sized.append(t)
        g = CompGraph(list(g.nodes), list(g.edges), sized)
    upd = [n.id for n in g.nodes if n.phase.value == "update"]
    per_upd = update_total * cost_scale / max(1, len(upd))
    nodes = []
    for n in g.nodes:
        if n.parameterized:
            nodes.append(n)
            continue
        c = costs.get(n.id)
        c = per_upd if n.id in upd else (c * cost_scale if c is not None else 0.0)
        nodes.append(replace(n, cost_hint=float(c)))
    tensors = [TensorSpec(t.id, t.producer, int(round(t.size_bytes * size_scale)), t.dtype) for t in g.tensors]
    return CompGraph(nodes, list(g.edges), tensors)


@dataclass
class LinkModel:
    """Rates (bytes/s) of the host link per direction and transfer path, and the
    wire/tensor ratio of each swapped tensor (graph tensor id -> ratio)."""

    d2h_ce: float
    h2d_ce: float
    d2h_zc: float
    h2d_zc: float
    overlap: bool = True
    wire_ratio: dict = field(default_factory=dict)
    zx_max_ratio: float = 0.92

    def rate(self, tid: int, d2h: bool) -> tuple[float, float]:
        """(wire bytes per tensor byte, bytes/s) of tensor tid's transfer."""
        r = self.wire_ratio.get(tid, 1.0)
        if r <= self.zx_max_ratio:
            return r, self.d2h_zc if d2h else self.h2d_zc
        return 1.0, self.d2h_ce if d2h else self.h2d_ce


def predict(g: CompGraph, link: LinkModel, order: dict | None = None, room_bytes: float = float("inf")) -> dict:
    """List-scheduling model of one step of rewritten graph ``g`` (see module doc).

    Memory is throttled like the pool throttles it: an op (or a swap-in's
    destination) that would take the live activations past ``room_bytes``
    waits until enough already-scheduled frees have happened — a tensor is
    released once all its readers finished, a swapped tensor only after its
    copy landed (sim.py:205-211).  ``fits`` is False when no pending free can
    make room (the real pool would raise LMS_OOM)."""
    import heapq

    order = order or topo_order(g)
    ex = _exec_set(g)
    seq = _schedule(g, order, ex)
    nbi, tbi = g.node_by_id, g.tensor_by_id

    def origin(tid):
        cur = tid
        while nbi[tbi[cur].producer].kind in (NodeKind.SWAP_OUT, NodeKind.SWAP_IN):
            ins = [e for e in g.in_edges(tbi[cur].producer) if e.action is EdgeAction.READ]
            if len(ins) != 1:
                break
            cur = ins[0].tensor
        return cur

    # readers per device-resident tensor (swap-outs read their source too)
    left, last = {}, {}
    for nid in seq:
        for e in g.in_edges(nid):
            if e.action is EdgeAction.READ and not nbi[tbi[e.tensor].producer].parameterized:
                left[e.tensor] = left.get(e.tensor, 0) + 1
    frees: list[tuple[float, int]] = []     # (time, bytes) of releases already known
    live = peak = 0
    fits = True
    stall = 0.0

    def make_room(t, need):
        """Earliest time >= t at which need bytes fit (pops the frees that happened).
        Queried on the compute stream's timeline only, which never goes back."""
        nonlocal live, fits, stall
        while frees and frees[0][0] <= t:
            live -= heapq.heappop(frees)[1]
        t_in = t
        while live + need > room_bytes:
            if not frees:
                fits = False
                break
            ft, b = heapq.heappop(frees)
            t = max(t, ft)
            live -= b
        stall += t - t_in
        return t

    start, finish = {}, {}
    engine = d2h = h2d = 0.0
    busy = {"d2h": 0.0, "h2d": 0.0}
    for nid in seq:
        node = nbi[nid]
        ready = 0.0
        reads = []
        for e in g.in_edges(nid):
            if e.action is EdgeAction.READ and not nbi[tbi[e.tensor].producer].parameterized:
                ready = max(ready, finish[tbi[e.tensor].producer])
                reads.append(e.tensor)
            elif e.action is EdgeAction.CONTROL and e.src in finish:
                ready = max(ready, finish[e.src])
        outs = [t for t in g.produced_tensors(nid) if t.size_bytes > 0]
        need = 0 if node.kind is NodeKind.SWAP_OUT else sum(t.size_bytes for t in outs)
        if node.kind is NodeKind.SWAP_OUT or node.kind is NodeKind.SWAP_IN:
            out_dir = node.kind is NodeKind.SWAP_OUT
            src = reads[0]
            ratio, bw = link.rate(origin(src), out_dir)
            dur = tbi[src].size_bytes * ratio / bw
            ch = d2h if (out_dir or not link.overlap) else h2d
            if out_dir:
                t0 = max(ch, ready)
            else:
                # the destination is allocated on the issuing (compute) thread, which
                # the pool blocks until the room is there; without a stall the H2D
                # starts when its control op (and swap-out) completed
                t_room = make_room(engine, need)
                stalled = t_room > engine
                engine = max(engine, t_room)
                t0 = max(ch, ready, t_room if stalled else 0.0)
            if out_dir or not link.overlap:
                d2h = t0 + dur
                if not link.overlap:
                    h2d = d2h
            else:
                h2d = t0 + dur
            busy["d2h" if out_dir else "h2d"] += dur
        else:
            t0 = make_room(max(engine, ready), need)
            dur = node.cost_hint
            engine = t0 + dur
        start[nid], finish[nid] = t0, t0 + dur
        live += need
        peak = max(peak, live)
        for tid in reads:
            last[tid] = max(last.get(tid, 0.0), finish[nid])
            left[tid] -= 1
            if left[tid] == 0:
                heapq.heappush(frees, (last[tid], tbi[tid].size_bytes))
        for t in outs:
            if node.kind is not NodeKind.SWAP_OUT and left.get(t.id, 0) == 0:
                heapq.heappush(frees, (finish[nid], t.size_bytes))   # only update edges read it
    makespan = max(finish.values(), default=0.0)
    return {"makespan": makespan, "peak_device_bytes": peak, "fits": fits, "alloc_stall": stall,
            "d2h_busy": busy["d2h"], "h2d_busy": busy["h2d"],
            "compute": sum(nbi[n].cost_hint for n in seq
                           if nbi[n].kind not in (NodeKind.SWAP_OUT, NodeKind.SWAP_IN))}


def plan_ranking(graph: CompGraph, cfgs, link: LinkModel, room_bytes: float):
    """Each config's predicted step under ``room_bytes`` of activation memory;
    those that fit come first, fastest first.  Returns [(cfg, prediction, fits)]."""
    from .rewriter import rewrite
    out = []
    for cfg in cfgs:
        g2, _ = rewrite(graph, cfg)
        p = predict(g2, link, room_bytes=room_bytes)
        out.append((cfg, p, p["fits"]))
    out.sort(key=lambda c: (not c[2], c[1]["makespan"]))
    return out
