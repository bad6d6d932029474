"""GPU executor for rewritten graphs in the interpreter vocabulary.

Replaces the reference's CPU executor ``interpret(g, inputs)``
(``interp.py:58-163``) and its modelled transfer engine / memory pool
(``simulate``, ``sim.py:139-476``) with the real thing on one B200:

* compute ops run on the caller's CUDA stream in the interpreter's serial
  (order, id) sequence — ``add/sub/mul/neg`` as elementwise kernels,
  ``matmul`` on cuBLAS (the only dense contraction), ``identity`` /
  ``assign_update`` / swap nodes as pass-throughs (interp.py:166-190);
* a ``swap_out`` node starts a D2H on liblms's copy channel the moment its
  producer is enqueued; the producer's block returns to the pool only after
  that copy completes (sim.py:205-211);
* a ``swap_in`` node is issued at its place in the serial order — right
  after its control predecessor (the op picked by lb/ub or chain_rule,
  rewriter.py:455-477) — so the H2D waits for that op's completion event and
  overlaps the ops in between; the consumer waits on the swap-in's event,
  not on the whole channel;
* every value is freed (stream-ordered) when its last reader is enqueued,
  so the pool's high-water mark is the measured ``peak_device_bytes``.

It returns the same ``{variable name: final value}`` map as ``interpret``
plus a *measured* :class:`~.report.SimReport`.  No CPU fallback: without
CUDA and liblms.so this raises.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

from .graph import CompGraph, EdgeAction, NodeKind, SWAP_KINDS, topo_order
from .report import SimReport, TraceEvent
from . import runtime as rt

_PASS_NAMES = ("identity", "assign_update")


@dataclass(frozen=True)
class ExecConfig:
    """Executor knobs.

    ``dtype`` is the arithmetic type on the GPU ("float32" per the north
    star; "float64" to compare with the fp64 reference at 1e-12).  ``codec``
    picks the swap transfer path (``ce`` copy engine, ``sm`` SM zero-copy,
    ``zvc`` lossless zero-value compression).  ``timing`` records transfer
    spans and swap-in stalls for the report.
    """

    device: int = 0
    dtype: str = "float32"
    codec: str = "ce"
    timing: bool = True
    return_numpy: bool = True


class _Swapped:
    """A swap-in destination that is valid once its H2D event has been waited on."""

    __slots__ = ("tensor", "handle", "waited")

    def __init__(self, tensor, handle):
        self.tensor = tensor
        self.handle = handle
        self.waited = False


def _origin(g: CompGraph, tid: int, memo: dict) -> int:
    path = []
    cur = tid
    while cur not in memo:
        path.append(cur)
        prod = g.node_by_id[g.tensor_by_id[cur].producer]
        if not (prod.kind in SWAP_KINDS or (prod.kind is NodeKind.COMPUTE and prod.name in _PASS_NAMES)):
            break
        reads = [e for e in g.in_edges(prod.id) if e.action is EdgeAction.READ]
        if len(reads) != 1 or reads[0].tensor in path:
            break
        cur = reads[0].tensor
    root = memo.get(cur, cur)
    for t in path:
        memo[t] = root
    return root


def _serial_schedule(g: CompGraph, order: dict[int, int]):
    """Runnable ops and their serial sequence (interp.py:84-158)."""
    starts = [n.id for n in g.nodes if n.parameterized]
    seen = set(starts)
    runnable: set[int] = set()
    stack = list(starts)
    while stack:
        for e in g.out_edges(stack.pop()):
            if e.action is EdgeAction.UPDATE or e.dst in seen:
                continue
            seen.add(e.dst)
            stack.append(e.dst)
            if not g.node_by_id[e.dst].parameterized:
                runnable.add(e.dst)
    pending = {}
    for nid in runnable:
        c = 0
        for e in g.in_edges(nid):
            if e.action is EdgeAction.READ:
                c += not g.node_by_id[g.tensor_by_id[e.tensor].producer].parameterized
            elif e.action is EdgeAction.CONTROL and e.src in runnable:
                c += 1
        pending[nid] = c
    heap = [(order[n], n) for n in runnable if pending[n] == 0]
    heapq.heapify(heap)
    seq = []
    while heap:
        _, nid = heapq.heappop(heap)
        seq.append(nid)
        wake = [e.dst for e in g.out_edges(nid) if e.action is EdgeAction.CONTROL and e.dst in runnable]
        for t in g.produced_tensors(nid):
            wake += [e.dst for e in g.consumer_edges(t.id) if e.action is EdgeAction.READ and e.dst in runnable]
        for d in wake:
            pending[d] -= 1
            if pending[d] == 0:
                heapq.heappush(heap, (order[d], d))
    if len(seq) != len(runnable):
        raise ValueError(f"ops never became ready (missing inputs?): {sorted(runnable - set(seq))}")
    return runnable, seq


def execute(g: CompGraph, inputs: dict, cfg: ExecConfig = ExecConfig(), ctx: rt.Context | None = None):
    """Run ``g`` once on the GPU; return (final variable states, measured SimReport)."""
    import torch

    if not torch.cuda.is_available():
        raise rt.LmsError("execute() needs a CUDA device; there is no CPU fallback")
    dev = torch.device("cuda", cfg.device)
    dtype = {"float32": torch.float32, "float64": torch.float64}[cfg.dtype]
    ctx = ctx or rt.installed_context()
    own_ctx = ctx is None
    if own_ctx:
        ctx = rt.Context(device=cfg.device, timing=cfg.timing)
    pool_measured = rt.installed_context() is ctx
    stream = torch.cuda.current_stream(dev)

    order = topo_order(g)
    runnable, seq = _serial_schedule(g, order)

    # bind parameterized nodes (interp.py:67-81)
    state = {}
    for n in g.nodes:
        if not n.parameterized:
            continue
        if n.name in inputs:
            v = inputs[n.name]
            state[n.id] = (v.to(device=dev, dtype=dtype) if torch.is_tensor(v)
                           else torch.as_tensor(v, dtype=dtype).to(dev))
        elif n.kind is NodeKind.CONSTANT:
            try:
                state[n.id] = torch.tensor(float(n.name), dtype=dtype, device=dev)
            except ValueError:
                raise ValueError(f"constant {n.name!r} (node {n.id}) is unbound "
                                 f"and its name is not a number") from None
        else:
            raise ValueError(f"variable {n.name!r} (node {n.id}) is unbound")

    # readers per tensor among runnable ops: a value is dropped after its last one
    readers: dict[int, int] = {}
    for nid in runnable:
        for e in g.in_edges(nid):
            if e.action is EdgeAction.READ:
                readers[e.tensor] = readers.get(e.tensor, 0) + 1

    torch.cuda.synchronize(dev)
    if pool_measured:
        ctx.reset_peaks()
        base_bytes = ctx.stats()["device_in_use"]
    else:
        torch.cuda.reset_peak_memory_stats(dev)
        base_bytes = torch.cuda.memory_allocated(dev)
    ctx.trace_clear()
    t_begin = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_begin.record(stream)

    memo: dict[int, int] = {}
    values: dict[int, object] = {}
    handles: dict[int, rt.SwapHandle] = {}   # swap_out output tensor -> host copy
    handle_uses: dict[int, int] = {}
    tensor_of_handle: dict[int, int] = {}
    waits_left: dict[int, int] = {}            # id(handle) -> swap-ins not yet waited on

    def take(e):
        prod = g.tensor_by_id[e.tensor].producer
        if g.node_by_id[prod].parameterized:
            return state[prod]
        v = values[e.tensor]
        if isinstance(v, _Swapped):
            if not v.waited:
                ctx.wait(v.handle, stream)
                v.waited = True
                key = id(v.handle)
                waits_left[key] -= 1
                if waits_left[key] == 0:
                    ctx.release(v.handle)  # last swap-in landed for this consumer side
            return v.tensor
        return v

    def consumed(e):
        left = readers[e.tensor] - 1
        readers[e.tensor] = left
        if left == 0:
            values.pop(e.tensor, None)  # stream-ordered free on the compute stream

    for nid in seq:
        node = g.node_by_id[nid]
        reads = sorted((e for e in g.in_edges(nid) if e.action is EdgeAction.READ),
                       key=lambda e: (_origin(g, e.tensor, memo), e.tensor))
        produced = g.produced_tensors(nid)
        if len(produced) > 1:
            raise ValueError(f"op {node.name!r} (node {nid}) has multiple outputs; "
                             "the interpreter vocabulary is single-output")
        if node.kind is NodeKind.SWAP_OUT:
            if len(reads) != 1:
                raise ValueError(f"'{node.name}' (node {nid}) expects 1 input(s), got {len(reads)}")
            src = take(reads[0])
            h = ctx.swap_out(src, cfg.codec, stream)
            consumed(reads[0])
            del src
            for t in produced:
                handles[t.id] = h
                handle_uses[t.id] = readers.get(t.id, 0)
                waits_left[id(h)] = readers.get(t.id, 0)
                tensor_of_handle[h.id] = _origin(g, t.id, memo)
            continue
        if node.kind is NodeKind.SWAP_IN:
            if len(reads) != 1:
                raise ValueError(f"'{node.name}' (node {nid}) expects 1 input(s), got {len(reads)}")
            src_t = reads[0].tensor
            h = handles[src_t]
            dst = ctx.swap_in(h, trigger_stream=stream)  # control op is already enqueued
            handle_uses[src_t] -= 1
            readers[src_t] -= 1
            for t in produced:
                values[t.id] = _Swapped(dst, h)
            continue
        args = [take(e) for e in reads]
        out = _apply(node, args, torch)
        for e in reads:
            consumed(e)
        del args
        for t in produced:
            values[t.id] = out
        for e in g.out_edges(nid):
            if e.action is not EdgeAction.UPDATE:
                continue
            var = g.node_by_id[e.dst]
            if not var.parameterized:
                raise ValueError(f"update edge into non-variable node {e.dst}")
            new = values[e.tensor]
            new = new.tensor if isinstance(new, _Swapped) else new
            if tuple(state[e.dst].shape) != tuple(new.shape):
                raise ValueError(f"update into {var.name!r}: shape {tuple(new.shape)} != "
                                 f"{tuple(state[e.dst].shape)}")
            state[e.dst] = new
        for t in produced:
            if readers.get(t.id, 0) == 0:
                values.pop(t.id, None)

    t_end.record(stream)
    for h in list(handles.values()):
        if not h.released:
            ctx.release(h)
    values.clear()
    torch.cuda.synchronize(dev)
    ctx.synchronize()

    st = ctx.stats()
    if pool_measured:
        peak = st["device_peak"] - base_bytes
    else:
        peak = torch.cuda.max_memory_allocated(dev) - base_bytes
    makespan = t_begin.elapsed_time(t_end) * 1e-3
    trace = []
    if cfg.timing:
        for x in ctx.trace():
            tid = tensor_of_handle.get(x["handle_id"])
            where = "host" if x["direction"] == 0 else f"acc:{cfg.device}"
            trace.append(TraceEvent(x["start_ms"] * 1e-3, "xfer_start", None, tid, x["wire_bytes"], where))
            trace.append(TraceEvent(x["end_ms"] * 1e-3, "xfer_finish", None, tid, x["wire_bytes"], where))
        trace.sort(key=lambda ev: ev.time)
    report = SimReport(
        peak_device_bytes=int(peak),
        peak_host_bytes=int(st["host_peak"]),
        makespan=makespan,
        transfer_time_total=(st["d2h_busy_ms"] + st["h2d_busy_ms"]) * 1e-3,
        transfer_wait_total=st["swap_wait_ms"] * 1e-3,
        oom=False,
        event_trace=trace,
    )
    out = {g.node_by_id[nid].name: v for nid, v in state.items()}
    if cfg.return_numpy:
        out = {k: v.double().cpu().numpy() for k, v in out.items()}
    if own_ctx:
        ctx.close()
    return out, report


def interpret(g: CompGraph, inputs: dict, ctx: rt.Context | None = None) -> dict:
    """Drop-in for the reference's ``interpret(g, inputs)`` (interp.py:58-163): the
    same ``{variable name: float64 ndarray}`` result, computed on the GPU in float64
    by :func:`execute` (swap nodes move real bytes through liblms)."""
    out, _ = execute(g, inputs, ExecConfig(dtype="float64", return_numpy=True), ctx=ctx)
    return out


def _apply(node, args, torch):
    name = node.name

    def arity(n):
        if len(args) != n:
            raise ValueError(f"{name!r} (node {node.id}) expects {n} input(s), got {len(args)}")

    if name in _PASS_NAMES:
        arity(1)
        return args[0]
    if name == "neg":
        arity(1)
        return torch.neg(args[0])
    if name in ("add", "sub", "mul"):
        arity(2)
        a, b = args
        if tuple(a.shape) != tuple(b.shape):
            raise ValueError(f"{name} (node {node.id}): shapes {tuple(a.shape)} and {tuple(b.shape)} differ")
        return {"add": torch.add, "sub": torch.sub, "mul": torch.mul}[name](a, b)
    if name == "matmul":
        arity(2)
        a, b = args
        if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[0]:
            raise ValueError(f"matmul (node {node.id}): shapes {tuple(a.shape)} @ {tuple(b.shape)} invalid")
        return torch.matmul(a, b)
    raise ValueError(f"unsupported op {name!r} (node {node.id})")
