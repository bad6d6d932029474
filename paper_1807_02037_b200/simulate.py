"""``simulate`` and ``free_step_oracle`` — the reference's sim.py surface, measured.

The reference models a rewritten step as a discrete-event simulation
(``swapgraph/sim.py:139-476``): ops allocate their outputs when they start,
drop inputs at refcount zero, swap nodes move ``size_bytes`` over modelled
D2H/H2D channels and the report gives peaks, makespan and transfer time.
Here the same schedule runs on the B200 through liblms:

* every tensor is a real block of ``size_bytes`` in the context's budgeted
  device pool (``SimConfig.device_capacity_bytes`` is the enforced budget on
  top of the permanently resident variables, sim.py:403-411);
* a compute op is one ``lms_sim_op`` launch on the compute stream: it checks
  each input word against the pattern its origin tensor was written with
  (a swap chain must deliver the producer's exact bytes), fills its outputs
  and lasts at least ``cost_hint * cost_unit_s`` seconds;
* a ``swap_out`` node is ``lms_swap_out`` on the D2H channel (the source block
  returns to the pool only after the copy lands, sim.py:205-211); a
  ``swap_in`` node allocates its destination and issues ``lms_swap_in`` on the
  H2D channel right after its control predecessor (rewriter.py:455-477);
  ``overlap_transfers=False`` puts both directions on one stream, the shared
  "xfer" channel (sim.py:284-290);
* the report has the reference's schema (sim.py:84-113) with measured values:
  pool high-water mark over the variables, pinned-pool high-water mark,
  CUDA-event makespan and copy-channel busy time, consumer stalls on
  swap-ins, and ``oom=True`` (instead of an exception) when the budget was
  exceeded — the run continues past the budget like the model does.

The link bandwidths in ``SimConfig`` are not modelled: the host link is real.
No CPU fallback: without CUDA and liblms.so this raises.
"""

from __future__ import annotations

import heapq

from .graph import HOST, CompGraph, EdgeAction, NodeKind, SWAP_KINDS, is_accelerator
from .report import SimConfig, SimReport, TraceEvent
from . import runtime as rt


def _exec_set(g: CompGraph) -> set[int]:
    """Ops reachable from the parameterized nodes over non-update edges
    (sim.py:124-134)."""
    seen = {n.id for n in g.nodes if n.parameterized}
    todo = list(seen)
    while todo:
        for e in g.out_edges(todo.pop()):
            if e.action is not EdgeAction.UPDATE and e.dst not in seen:
                seen.add(e.dst)
                todo.append(e.dst)
    return {nid for nid in seen if not g.node_by_id[nid].parameterized}


def free_step_oracle(g: CompGraph, order: dict[int, int], tensor_id: int) -> int:
    """Order step at which ``tensor_id``'s refcount reaches zero in a serial run
    (sim.py:479-508): reachable ops run in ascending (order, id); each executed
    consumer drops its read references, update edges drop theirs when the
    producer itself runs.  The pool's free policy; equals γ(producer) +
    lifetime (test_acceptance.py:142-164)."""
    t = g.tensor_by_id[tensor_id]
    ex = _exec_set(g)
    cons = g.consumer_edges(tensor_id)
    per_reader: dict[int, int] = {}
    for e in cons:
        if e.action is EdgeAction.READ and e.dst in ex:
            per_reader[e.dst] = per_reader.get(e.dst, 0) + 1
    n_upd = sum(1 for e in cons if e.action is EdgeAction.UPDATE)
    left = sum(per_reader.values()) + n_upd
    birth = order[t.producer]
    if left == 0:
        return birth
    for nid in sorted(ex, key=lambda n: (order[n], n)):
        if nid == t.producer:
            left -= n_upd
            if left <= 0:
                return birth
        k = per_reader.get(nid)
        if k:
            left -= k
            if left <= 0:
                return order[nid]
    return max((order[n] for n in per_reader), default=birth)


def _schedule(g: CompGraph, order: dict[int, int], ex: set[int]) -> list[int]:
    """Issue sequence: ready ops in (order, id) as their read and control
    predecessors are issued (one engine per device, sim.py:325-354)."""
    pending = {}
    for nid in ex:
        c = 0
        for e in g.in_edges(nid):
            if e.action is EdgeAction.READ:
                c += not g.node_by_id[g.tensor_by_id[e.tensor].producer].parameterized
            elif e.action is EdgeAction.CONTROL and e.src in ex:
                c += 1
        pending[nid] = c
    heap = [(order[n], n) for n in ex if pending[n] == 0]
    heapq.heapify(heap)
    seq = []
    while heap:
        _, nid = heapq.heappop(heap)
        seq.append(nid)
        wake = [e.dst for e in g.out_edges(nid) if e.action is EdgeAction.CONTROL and e.dst in ex]
        for t in g.produced_tensors(nid):
            wake += [e.dst for e in g.consumer_edges(t.id) if e.action is EdgeAction.READ and e.dst in ex]
        for d in wake:
            pending[d] -= 1
            if pending[d] == 0:
                heapq.heappush(heap, (order[d], d))
    if len(seq) != len(ex):
        blocked = sorted(ex - set(seq))
        from .report import DeadlockError
        raise DeadlockError("simulation stalled; nodes never ready: " + ", ".join(map(str, blocked[:8])))
    return seq


def _round_block(n: int) -> int:
    # the device pool's block granularity: 512 B up to 1 MiB, 2 MiB above
    if n <= 1 << 20:
        return max(512, (n + 511) // 512 * 512)
    return (n + (2 << 20) - 1) // (2 << 20) * (2 << 20)


class _SwapIn:
    __slots__ = ("ptr", "handle", "waited")

    def __init__(self, ptr, handle):
        self.ptr, self.handle, self.waited = ptr, handle, False


def simulate(g: CompGraph, order: dict[int, int], cfg: SimConfig = SimConfig(), *, device: int = 0,
             cost_unit_s: float = 0.0, verify: bool = True) -> SimReport:
    """Run the schedule of ``g`` on the GPU and report what was measured
    (sim.py:139 signature; extension keywords: ``cost_unit_s`` = seconds per
    unit of ``cost_hint``, ``verify`` = fail if a swap chain delivered wrong
    bytes)."""
    import torch

    ex = _exec_set(g)
    for t in g.tensors:
        p = g.node_by_id[t.producer]
        if (p.parameterized or t.producer in ex) and t.size_bytes <= 0:
            raise ValueError(f"tensor {t.id} participates in simulation but has size_bytes={t.size_bytes}")
    accs = {g.node_by_id[n].device for n in ex if g.node_by_id[n].kind not in SWAP_KINDS}
    accs |= {n.device for n in g.nodes if n.parameterized}
    if len(accs) > 1 or any(not is_accelerator(d) for d in accs):
        raise ValueError(f"the measured simulate runs one accelerator plus host swap nodes; devices {sorted(accs)}")
    if any(g.node_by_id[n].device != HOST for n in ex if g.node_by_id[n].kind in SWAP_KINDS):
        raise ValueError("swap nodes must be host-placed (graph.py: swap-off-host)")
    if not torch.cuda.is_available():
        raise rt.LmsError("simulate() measures on a CUDA device; there is no CPU fallback")
    seq = _schedule(g, order, ex)

    # every block the run can hold at once is at most every tensor it makes
    var_bytes = sum(_round_block(t.size_bytes) for n in g.nodes if n.parameterized
                    for t in g.produced_tensors(n.id))
    run_bytes = sum(_round_block(t.size_bytes) for n in ex for t in g.produced_tensors(n)
                    if g.node_by_id[n].kind is not NodeKind.SWAP_OUT)
    base_bytes = var_bytes + 512   # + the verification counter
    reserve = base_bytes + run_bytes + (64 << 20)
    dev = torch.device("cuda", device)
    ctx = rt.Context(device=device, device_reserve=reserve, host_chunk=max(64 << 20, min(run_bytes, 1 << 30)),
                     overlap_transfers=cfg.overlap_transfers, timing=True)
    stream = torch.cuda.current_stream(dev)
    oom = False
    try:
        ctx.set_limit(min(reserve, base_bytes + cfg.device_capacity_bytes))

        def alloc(nbytes):
            nonlocal oom
            try:
                return ctx.dev_alloc(nbytes, stream)
            except rt.LmsOutOfMemoryError:
                oom = True        # the model reports oom and runs on (sim.py:471)
                ctx.set_limit(reserve)
                return ctx.dev_alloc(nbytes, stream)

        errors = ctx.dev_alloc(4, stream)
        torch.cuda.synchronize(dev)
        err_view = torch.as_tensor(rt.DeviceBuffer(errors, 4), device=dev)
        err_view.zero_()
        state = {}
        for n in g.nodes:
            if n.parameterized:
                for t in g.produced_tensors(n.id):
                    state[t.id] = ctx.dev_alloc(t.size_bytes, stream)
                    ctx.sim_op([(state[t.id], t.size_bytes, t.id)], [], errors, 0, stream)
        readers: dict[int, int] = {}
        for nid in ex:
            for e in g.in_edges(nid):
                if e.action is EdgeAction.READ:
                    readers[e.tensor] = readers.get(e.tensor, 0) + 1
        origin: dict[int, int] = {}

        def origin_of(tid):
            cur = tid
            while True:
                prod = g.node_by_id[g.tensor_by_id[cur].producer]
                if prod.kind not in SWAP_KINDS:
                    break
                ins = [e for e in g.in_edges(prod.id) if e.action is EdgeAction.READ]
                if len(ins) != 1:
                    break
                cur = ins[0].tensor
            origin[tid] = cur
            return cur

        torch.cuda.synchronize(dev)
        ctx.synchronize()
        ctx.trace_clear()
        ctx.reset_peaks()
        t_begin = torch.cuda.Event(enable_timing=True)
        t_begin.record(stream)
        values: dict[int, object] = {}
        handles: dict[int, rt.SwapHandle] = {}
        waits_left: dict[int, int] = {}
        op_events = []
        spin = max(0.0, cost_unit_s)

        def read(e):
            prod = g.node_by_id[g.tensor_by_id[e.tensor].producer]
            if prod.parameterized:
                return state[e.tensor]
            v = values[e.tensor]
            if isinstance(v, _SwapIn):
                if not v.waited:
                    ctx.wait(v.handle, stream)
                    v.waited = True
                    waits_left[v.handle.id] -= 1
                    if waits_left[v.handle.id] == 0:
                        ctx.release(v.handle)
                return v.ptr
            return v

        def consumed(tid):
            readers[tid] -= 1
            if readers[tid] == 0:
                v = values.pop(tid, None)
                if isinstance(v, _SwapIn):
                    v = v.ptr
                if isinstance(v, int):
                    ctx.dev_free(v, stream)

        for nid in seq:
            node = g.node_by_id[nid]
            reads = [e for e in g.in_edges(nid) if e.action is EdgeAction.READ]
            produced = g.produced_tensors(nid)
            if node.kind is NodeKind.SWAP_OUT:
                (e,) = reads
                src = read(e)
                h = ctx.swap_out_raw(src, g.tensor_by_id[e.tensor].size_bytes, "ce", stream)
                consumed(e.tensor)
                for t in produced:
                    handles[t.id] = h
                    waits_left[h.id] = readers.get(t.id, 0)
                    if readers.get(t.id, 0) == 0:
                        ctx.release(h)
                continue
            if node.kind is NodeKind.SWAP_IN:
                (e,) = reads
                h = handles[e.tensor]
                for t in produced:
                    dst = alloc(t.size_bytes)
                    ctx.swap_in_raw(h, dst, trigger_stream=stream)
                    values[t.id] = _SwapIn(dst, h)
                    if readers.get(t.id, 0) == 0:
                        ctx.wait(h, stream)
                        ctx.dev_free(dst, stream)
                        values.pop(t.id)
                readers[e.tensor] -= 1
                continue
            ins = [(read(e), g.tensor_by_id[e.tensor].size_bytes, origin.get(e.tensor) or origin_of(e.tensor))
                   for e in reads]
            outs = []
            for t in produced:
                values[t.id] = alloc(t.size_bytes)
                outs.append((values[t.id], t.size_bytes, t.id))
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            ctx.sim_op(outs, ins, errors, int(node.cost_hint * spin * 1e9), stream)
            ev1.record(stream)
            op_events.append((nid, ev0, ev1))
            for e in reads:
                if not g.node_by_id[g.tensor_by_id[e.tensor].producer].parameterized:
                    consumed(e.tensor)
            for t in produced:
                if readers.get(t.id, 0) == 0:   # only update edges: committed at completion
                    ctx.dev_free(values.pop(t.id), stream)
        for h in handles.values():
            if not h.released:
                ctx.release(h)
        d2h, h2d = ctx.streams()
        stream.wait_stream(d2h)
        stream.wait_stream(h2d)
        t_end = torch.cuda.Event(enable_timing=True)
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        ctx.synchronize()
        bad = int(err_view.cpu().view(torch.int32).item())
        if verify and bad:
            raise rt.LmsError(f"simulate: {bad} words differed from their producers' (a swap chain "
                              f"delivered wrong bytes)")
        st = ctx.stats()
        trace = []
        for nid, a, b in op_events:
            where = g.node_by_id[nid].device
            trace.append(TraceEvent(t_begin.elapsed_time(a) * 1e-3, "start", nid, None, 0, where))
            trace.append(TraceEvent(t_begin.elapsed_time(b) * 1e-3, "finish", nid, None, 0, where))
        tensor_of = {h.id: origin_of(k) for k, h in handles.items()}
        for x in ctx.trace():
            tid = tensor_of.get(x["handle_id"])
            where = HOST if x["direction"] == 0 else next(iter(accs))
            trace.append(TraceEvent(x["start_ms"] * 1e-3, "xfer_start", None, tid, x["wire_bytes"], where))
            trace.append(TraceEvent(x["end_ms"] * 1e-3, "xfer_finish", None, tid, x["wire_bytes"], where))
        trace.sort(key=lambda ev: ev.time)
        return SimReport(
            peak_device_bytes=int(st["device_peak"] - base_bytes),
            peak_host_bytes=int(st["host_peak"]),
            makespan=t_begin.elapsed_time(t_end) * 1e-3,
            transfer_time_total=(st["d2h_busy_ms"] + st["h2d_busy_ms"]) * 1e-3,
            transfer_wait_total=st["swap_wait_ms"] * 1e-3,
            oom=oom or st["device_peak"] - base_bytes > cfg.device_capacity_bytes,
            event_trace=trace,
        )
    finally:
        torch.cuda.synchronize(dev)
        ctx.close()
