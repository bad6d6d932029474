"""PyTorch training steps under TFLMS swapping.

This is the caller side of the rewrite: it captures a
training step as a :class:`~.graph.CompGraph`, runs the unchanged
:func:`~.rewriter.rewrite` on it, and executes the rewritten schedule with
liblms:

capture   one traced step records every tensor autograd saves for backward
          (``saved_tensors_hooks`` pack calls, in order) and, in backward,
          which autograd node consumed it (``torch._C._current_autograd_node``).
          The graph has a forward op F(n) and a backward op B(n) per autograd
          node n (creation order = ``_sequence_nr``), a variable per parameter
          and per step input, and one update op per parameter.  Saved tensors
          become F(producer) -> B(consumer) read edges — the paper's
          forward->backward candidates (PAPER §4.1, rewriter.py:214-238).
rewrite   the reference algorithm, any ``RewriteConfig`` (n_tensors, lb/ub,
          chain_rule/direct_order, fuse_swapins, incl/excl types ...).
execute   pack hook = swap-out: the first pack of a selected tensor starts a
          D2H on liblms's copy channel (fused swap-outs: one per tensor,
          rewriter.py:294-334) and autograd keeps only a handle, so the
          device block returns to the budgeted pool once the D2H is done.
          Each swap-in group (one rewritten swap-in node; fused groups feed
          several consumers) is issued by a post-hook on its control op's
          autograd node, so the H2D starts when that op finishes; the unpack
          hook only makes the consumer's stream wait on the group's event.

Conventions kept from the reference: swap-ins with no control op are issued
eagerly right after their swap-out (rewriter.py:472-475); control ops that
fall in the forward phase fire at the start of backward (an autograd node
cannot be hooked on its forward execution).
"""

from __future__ import annotations

import contextlib
import time
from dataclasses import dataclass, field

import torch
from torch.overrides import TorchFunctionMode
from torch.utils._pytree import tree_flatten

from .graph import (
    CompGraph,
    EdgeAction,
    EdgeRec,
    NodeKind,
    OpNode,
    Phase,
    TensorSpec,
    compute_node,
    variable_node,
)
from .rewriter import RewriteConfig, RewriteReport, rewrite
from . import runtime as rt

_current_node = torch._C._current_autograd_node


def _fwd_name(node) -> str:
    n = node.name()
    for suffix in ("Backward0", "Backward1", "Backward"):
        if n.endswith(suffix):
            return n[: -len(suffix)]
    return n


def _walk(root):
    """Every autograd node reachable from ``root`` (BFS over next_functions)."""
    seen = {}
    todo = [root]
    while todo:
        n = todo.pop()
        if n is None or n in seen:
            continue
        seen[n] = True
        for nxt, _ in n.next_functions:
            if nxt is not None and nxt not in seen:
                todo.append(nxt)
    return list(seen)


def _is_accumulate(node) -> bool:
    return node.name() == "torch::autograd::AccumulateGrad"


@dataclass
class _Saved:
    """One distinct saved tensor seen at capture."""

    tid: int
    nbytes: int
    producer: object            # autograd node, "self" (saved by its own op) or None (leaf)
    is_param: bool
    packs: list = field(default_factory=list)   # pack indices that saved it
    zero_frac: float = 0.0
    zx_ratio: float = 1.0


@dataclass
class SwapGroup:
    """One swap-in node of the rewritten graph."""

    gid: int
    saved: int                  # index into plan.saved
    packs: list                 # pack indices this group serves
    trigger: int | None         # node rank of the control op's node; None = eager
    trigger_kind: str           # "backward" | "forward->bwd-start" | "eager" | "forward"
    node: int = -1              # the swap-in node's id in the rewritten graph
    # forward-side swap-ins (swap_branches: fwd->fwd edges, rewriter.py:231)
    fwd_consumers: tuple = ()   # node ranks of the forward ops reading the swapped-in tensor
    tensor: int = -1            # the captured graph's tensor id
    producer_rank: int = -1     # node rank of the tensor's producer
    release_rank: int = -1      # last forward op still reading the device copy
    nbytes: int = 0


@dataclass
class SwapPlan:
    """Everything the executor needs, keyed by pack index and node rank."""

    graph: CompGraph
    rewritten: CompGraph
    report: RewriteReport
    n_packs: int
    pack_saved: list            # pack idx -> saved index (or -1 if kept)
    saved: list                 # list[_SavedInfo]
    groups: list                # list[SwapGroup]
    pack_group: dict            # pack idx -> group id
    triggers: dict              # node rank -> [group ids]
    bwd_start_groups: list
    eager_groups: list
    swapped_bytes_per_step: int
    saved_bytes_per_step: int
    capture_batch: int
    rewrite_seconds: float
    fwd_groups: list = field(default_factory=list)      # forward-side swap-in groups
    fwd_triggers: dict = field(default_factory=dict)    # forward node rank -> [group ids]

    def summary(self) -> dict:
        return {
            "tensors_saved": len(self.saved),
            "tensors_swapped": self.report.tensors_swapped,
            "swap_ins": len(self.groups),
            "control_edges": self.report.control_edges_added,
            "eager_swap_ins": len(self.eager_groups),
            "forward_swap_ins": len(self.fwd_groups),
            "bwd_start_swap_ins": len(self.bwd_start_groups),
            "swapped_bytes_capture": self.swapped_bytes_per_step,
            "saved_bytes_capture": self.saved_bytes_per_step,
            "graph_nodes": len(self.graph.nodes),
            "rewrite_seconds": self.rewrite_seconds,
        }


@dataclass
class _SavedInfo:
    tid: int
    nbytes: int
    swapped: bool
    zero_frac: float = 0.0
    zx_ratio: float = 1.0


def zx_ratio_estimate(t, max_words: int = 1 << 18) -> float:
    """Wire bytes / tensor bytes the ZX codec (ZVC v3 with exponent planes,
    kernels.cuh) would need, computed with the codec's own per-tile rules on
    the tensor's first ``max_words`` 32-bit words (whole 4096-word tiles; one
    host copy of the sample, numpy on the host: no per-tensor kernel chain)."""
    import numpy as np
    if not t.numel() or t.element_size() != 4 or not t.is_contiguous():
        return 1.0
    w = t.detach().reshape(-1).view(torch.int32)
    n = min(w.numel(), max_words) // 4096 * 4096
    if n == 0:
        return 1.0
    x = w[:n].cpu().numpy().view(np.uint32).reshape(-1, 4096)
    nz = x != 0
    e7 = ((x >> 24) & 0x7F).astype(np.int64)
    s = (x >> 31).astype(np.int64)
    cnt = nz.sum(1)

    def pad16(v):
        return (v + 15) // 16 * 16

    def bits(r):
        return np.where(r > 0, np.floor(np.log2(np.maximum(r, 1))) + 1, 0)

    raw = np.full(cnt.shape, 16384.0)
    mask = 512.0 + pad16(4 * cnt)
    kd = bits(e7.max(1) - e7.min(1))
    sd = (s.max(1) != s.min(1)).astype(np.float64)
    expd = 96.0 * 128 + pad16(4 * 128 * (kd + sd))
    km = bits(np.where(nz, e7, 0).max(1) - np.where(nz, e7, 127).min(1))
    sm = (np.where(nz, s, 0).max(1) != np.where(nz, s, 1).min(1)).astype(np.float64)
    expm = np.where(cnt > 0, 512.0 + pad16(3 * cnt) + pad16(np.ceil(cnt * (km + sm) / 8)), mask)
    best = np.minimum(np.minimum(raw, mask), np.minimum(expd, expm))
    return float((best.sum() + 8 * best.size) / (4.0 * n))


class _Capture:
    """Records packs (forward) and consumers (backward) for one traced step."""

    def __init__(self, min_bytes: int = 0):
        self.packs = []        # pack idx -> (tensor key, nbytes, grad_fn or None, is_leaf, requires_grad)
        self.keep = []         # strong refs so addresses stay unique during capture
        self.consumer = {}     # pack idx -> autograd node that unpacked it
        self.zero_frac = []    # pack idx -> share of zero words (capture-time contents)
        self.zx_ratio = []     # pack idx -> ZX codec wire/tensor bytes (capture-time contents)
        self.min_bytes = min_bytes   # smaller tensors are never swap candidates: not measured
        self._measured = {}    # tensor key -> (zero_frac, zx_ratio): a tensor saved twice is measured once

    def pack(self, t):
        k = len(self.packs)
        key = (t.data_ptr(), tuple(t.shape), tuple(t.stride()), t.dtype)
        nbytes = t.numel() * t.element_size()
        is_param = isinstance(t, torch.nn.Parameter)
        self.packs.append((key, nbytes, t.grad_fn, t.is_leaf, t.requires_grad, is_param))
        m = self._measured.get(key)
        if m is None:
            # share of all-zero 32-bit words, and the ZX codec's stream ratio
            zf, zx = 0.0, 1.0
            if (nbytes >= self.min_bytes and t.numel() and t.element_size() == 4 and t.is_contiguous()
                    and not is_param):
                w = t.detach().view(-1).view(torch.int32)
                if w.numel() > (1 << 22):      # a strided sample: no tensor-sized temporaries
                    w = w[:: w.numel() >> 22]
                zf = 1.0 - float(torch.count_nonzero(w)) / w.numel()
                zx = zx_ratio_estimate(t)
            m = self._measured[key] = (zf, zx)
        self.zero_frac.append(m[0])
        self.zx_ratio.append(m[1])
        t = t.detach()   # no tensor -> grad_fn -> saved -> tensor cycle (see SwapExecutor.pack)
        self.keep.append(t)
        return (k, t)

    def unpack(self, packed):
        k, t = packed
        if k not in self.consumer:
            self.consumer[k] = _current_node()
        return t


class _OutputBytes(TorchFunctionMode):
    """Capture: bytes of every autograd node's forward output, so forward->forward
    edges (the paper's branch tensors, e.g. U-Net skips) carry real sizes."""

    def __init__(self):
        super().__init__()
        self.nbytes = {}
        self.first = None

    def __torch_function__(self, func, types, args=(), kwargs=None):
        out = func(*args, **(kwargs or {}))
        for t in tree_flatten(out)[0]:
            if isinstance(t, torch.Tensor) and t.grad_fn is not None:
                gf = t.grad_fn
                if self.first is None:
                    self.first = gf
                nb = t.numel() * t.element_size()
                if nb > self.nbytes.get(gf, -1):
                    self.nbytes[gf] = nb
        return out


def capture_graph(forward_fn, min_swap_bytes: int = 1 << 16, persistent=()):
    """Trace one step — ``forward_fn()`` returns the loss, backward runs here — into a CompGraph.

    ``persistent``: tensors that outlive the step (parameters, buffers, the
    step's inputs); saved references to them become variable reads and are
    never swapped.  Any other saved tensor without a ``grad_fn`` (pooling
    indices, saved batch statistics, workspaces) is an output of the op that
    saves it.  Returns (graph, meta) where meta maps graph ids back to pack
    indices and autograd-node ranks.  The traced step's gradients are left in
    place.
    """
    keep_ptrs = {t.data_ptr() for t in persistent if t is not None and t.numel()}
    cap = _Capture(min_swap_bytes)
    sizes = _OutputBytes()
    with torch.autograd.graph.saved_tensors_hooks(cap.pack, cap.unpack), sizes:
        loss = forward_fn()
    root = loss.grad_fn
    nodes = _walk(root)
    loss.backward()
    if torch.cuda.is_available():
        torch.cuda.synchronize()

    accs = [n for n in nodes if _is_accumulate(n)]
    ops = sorted((n for n in nodes if not _is_accumulate(n)), key=lambda n: n._sequence_nr())
    seq0 = ops[0]._sequence_nr() if ops else 0
    rank = {n: n._sequence_nr() - seq0 for n in ops}

    # ids: variables first (params in pack/encounter order, then inputs), then F, B, U ops
    gnodes, gedges, gtensors = [], [], []

    def new_tensor(producer_id, nbytes):
        tid = len(gtensors)
        gtensors.append(TensorSpec(tid, producer_id, int(nbytes)))
        return tid

    var_of_acc = {}
    for i, a in enumerate(accs):
        nid = len(gnodes)
        gnodes.append(variable_node(nid, f"param_{i}", scope="params"))
        var_of_acc[a] = (nid, new_tensor(nid, 0))
    input_var = len(gnodes)
    gnodes.append(variable_node(input_var, "input", scope="inputs"))
    input_t = new_tensor(input_var, 0)
    seed_var = len(gnodes)
    gnodes.append(variable_node(seed_var, "grad_seed", scope="inputs"))
    seed_t = new_tensor(seed_var, 0)

    F, B = {}, {}
    main_out = {}
    for n in ops:
        nid = len(gnodes)
        gnodes.append(compute_node(nid, _fwd_name(n), scope="model", phase=Phase.FORWARD))
        F[n] = nid
        main_out[n] = new_tensor(nid, 0)
    for n in ops:
        for nxt, _ in n.next_functions:
            if nxt is None:
                gedges.append(EdgeRec(input_var, F[n], EdgeAction.READ, input_t))
            elif _is_accumulate(nxt):
                v, vt = var_of_acc[nxt]
                gedges.append(EdgeRec(v, F[n], EdgeAction.READ, vt))
            else:
                gedges.append(EdgeRec(F[nxt], F[n], EdgeAction.READ, main_out[nxt]))
        if not n.next_functions:
            gedges.append(EdgeRec(input_var, F[n], EdgeAction.READ, input_t))

    # distinct saved tensors; producer = grad_fn, or the saving op itself for
    # non-differentiable outputs (indices, saved statistics)
    by_key = {}
    saved = []
    pack_saved = []
    for k, (key, nbytes, grad_fn, is_leaf, req, is_param) in enumerate(cap.packs):
        consumer = cap.consumer.get(k)
        if consumer is None or consumer not in rank:
            pack_saved.append(-1)
            continue
        s = by_key.get(key)
        if s is None:
            if is_param or (is_leaf and req) or key[0] in keep_ptrs:
                producer = None   # parameter, buffer or step input: a variable
            elif grad_fn is not None and grad_fn in rank:
                producer = grad_fn
            else:
                producer = "self"  # non-differentiable output of the saving op
            s = _Saved(len(saved), nbytes, producer, is_param, zero_frac=cap.zero_frac[k],
                       zx_ratio=cap.zx_ratio[k])
            by_key[key] = s
            saved.append(s)
        s.packs.append(k)
        pack_saved.append(s.tid)

    for n in reversed(ops):  # backward ops in reverse creation order
        nid = len(gnodes)
        gnodes.append(compute_node(nid, n.name(), scope="grads", phase=Phase.BACKWARD))
        B[n] = nid
    grad_out = {n: new_tensor(B[n], 0) for n in ops}
    if root in B:
        gedges.append(EdgeRec(seed_var, B[root], EdgeAction.READ, seed_t))
    acc_grad = {}
    for n in ops:
        for nxt, _ in n.next_functions:
            if nxt is None:
                continue
            if _is_accumulate(nxt):
                acc_grad.setdefault(nxt, []).append(n)
            else:
                gedges.append(EdgeRec(B[n], B[nxt], EdgeAction.READ, grad_out[n]))

    saved_tensor_id = {}
    seen_edge = set()
    self_prod = {}  # saved index -> op that produced a grad_fn-less tensor (its first saver)
    for k, si in enumerate(pack_saved):
        if si < 0:
            continue
        s = saved[si]
        cons = cap.consumer[k]
        if s.producer is None:
            continue  # params and inputs stay resident (variables are never swapped)
        prod = self_prod.setdefault(si, cons) if s.producer == "self" else s.producer
        if s.producer != "self" and s.nbytes == 0:
            continue
        tid = saved_tensor_id.get(si)
        if tid is None:
            if s.producer != "self" and prod in main_out and gtensors[main_out[prod]].size_bytes == 0:
                tid = main_out[prod]
                gtensors[tid] = TensorSpec(tid, F[prod], s.nbytes)
            else:
                tid = new_tensor(F[prod], s.nbytes)
            saved_tensor_id[si] = tid
        if s.nbytes < min_swap_bytes:
            continue  # tiny tensors stay on the device; no candidate edge
        e = EdgeRec(F[prod], B[cons], EdgeAction.READ, tid)
        if e not in seen_edge:
            seen_edge.add(e)
            gedges.append(e)

    # forward outputs nobody saved: their fwd->fwd edges carry the output's bytes
    for n in ops:
        tid = main_out[n]
        if gtensors[tid].size_bytes == 0 and sizes.nbytes.get(n, 0) > 0:
            gtensors[tid] = TensorSpec(tid, F[n], sizes.nbytes[n])

    for a, users in acc_grad.items():
        v, vt = var_of_acc[a]
        uid = len(gnodes)
        gnodes.append(compute_node(uid, "sgd", scope="optimizer", phase=Phase.UPDATE))
        gedges.append(EdgeRec(v, uid, EdgeAction.READ, vt))
        for u in users:
            gedges.append(EdgeRec(B[u], uid, EdgeAction.READ, grad_out[u]))
        upd = new_tensor(uid, 0)
        gedges.append(EdgeRec(uid, v, EdgeAction.UPDATE, upd))

    g = CompGraph(gnodes, gedges, gtensors)
    meta = {
        "n_packs": len(cap.packs),
        "pack_saved": pack_saved,
        "saved": saved,
        "saved_tensor_id": saved_tensor_id,
        "F": {F[n]: rank[n] for n in ops},
        "B": {B[n]: rank[n] for n in ops},
        "consumer_rank": {k: rank.get(c) for k, c in cap.consumer.items()},
        "min_swap_bytes": min_swap_bytes,
        # forward-side swaps find op outputs by their node's rank counted from
        # the first node the forward creates; that must be rank 0 here
        "fwd_ranks_ok": sizes.first is not None and rank.get(sizes.first) == 0,
    }
    return g, meta


def build_plan(g: CompGraph, meta: dict, cfg: RewriteConfig, capture_batch: int,
               far_cfg: RewriteConfig | None = None, far_max_fraction: float = 0.0) -> SwapPlan:
    """Rewrite the captured graph and map swap-ins back onto pack indices / nodes.

    ``far_cfg`` (an extension, not in the reference): a second rewrite of the
    same graph with only the control-op window changed (e.g. a larger lb);
    swap-ins of tensors smaller than ``far_max_fraction`` x the largest swapped
    tensor take their control op from it.  Both rewrites insert the same
    swap nodes; small tensors start their H2D further ahead of the consumer,
    big ones keep the memory-lean window.
    """
    t0 = time.perf_counter()
    out, rep = rewrite(g, cfg)
    far_ctrl = {}
    if far_cfg is not None and far_max_fraction > 0:
        far_out, _ = rewrite(g, far_cfg)
        ids = {n.id for n in out.nodes if n.kind is NodeKind.SWAP_IN}
        far_ids = {n.id for n in far_out.nodes if n.kind is NodeKind.SWAP_IN}
        if ids != far_ids:
            raise ValueError("far_cfg must differ from cfg only in the control-op window "
                             "(lb/ub/ctrld_strategy): its swap-ins differ")
        far_ctrl = {e.dst: e.src for e in far_out.edges if e.action is EdgeAction.CONTROL}
    dt = time.perf_counter() - t0
    tid_to_saved = {tid: si for si, tid in meta["saved_tensor_id"].items()}
    B = meta["B"]
    F = meta["F"]
    swapped_tids = {tid for _, _, tid in rep.edges_rewritten}
    pack_saved = meta["pack_saved"]
    saved_info = [_SavedInfo(s.tid, s.nbytes, meta["saved_tensor_id"].get(s.tid) in swapped_tids,
                             s.zero_frac, s.zx_ratio) for s in meta["saved"]]

    # swap-in nodes -> groups
    groups = []
    pack_group = {}
    triggers: dict[int, list] = {}
    bwd_start, eager = [], []
    fwd_groups, fwd_triggers = [], {}
    ctrl_of = {e.dst: e.src for e in out.edges if e.action is EdgeAction.CONTROL}
    biggest = max((s.nbytes for s in saved_info if s.swapped), default=0)
    for n in out.nodes:
        if n.kind is not NodeKind.SWAP_IN:
            continue
        src = next(e for e in out.in_edges(n.id) if e.action is EdgeAction.READ)
        so = src.src
        orig = next(e for e in out.in_edges(so) if e.action is EdgeAction.READ).tensor
        si = tid_to_saved.get(orig)
        dsts = [e.dst for e in out.out_edges(n.id) if e.action is EdgeAction.READ]
        bwd_cons = {B[d] for d in dsts if d in B}
        fwd_cons = sorted(F[d] for d in dsts if d in F)
        c = ctrl_of.get(n.id)
        if fwd_cons:
            # a branch swap (fwd->fwd, rewriter.py:231): the forward pass itself
            # frees the device copy and restores it before the consumer
            grp = _forward_group(out, meta, n.id, orig, si, fwd_cons, c, len(groups) + len(fwd_groups))
            if grp is not None:
                fwd_groups.append(grp)
                if grp.trigger_kind == "forward":
                    fwd_triggers.setdefault(grp.trigger, []).append(grp.gid)
            if not bwd_cons:
                continue
        if si is None:
            continue
        packs = [k for k in meta["saved"][si].packs if meta["consumer_rank"].get(k) in bwd_cons]
        if far_ctrl and meta["saved"][si].nbytes < far_max_fraction * biggest and n.id in far_ctrl:
            c = far_ctrl[n.id]
        if c is None:
            kind, trig = "eager", None
        elif c in B:
            kind, trig = "backward", B[c]
        else:
            kind, trig = "forward->bwd-start", None
        grp = SwapGroup(len(groups) + len(fwd_groups), si, packs, trig, kind, n.id)
        groups.append(grp)
        for k in packs:
            pack_group[k] = grp.gid
        if kind == "backward":
            triggers.setdefault(trig, []).append(grp.gid)
        elif kind == "eager":
            eager.append(grp.gid)
        else:
            bwd_start.append(grp.gid)
    # group ids index plan.groups: forward groups take their slots after renumbering
    allg = sorted(groups + fwd_groups, key=lambda g: g.gid)
    assert [g.gid for g in allg] == list(range(len(allg)))
    groups = allg
    # packs of a swapped tensor whose consumer edge was not rewritten keep the tensor
    pack_is_swapped = [k in pack_group for k in range(meta["n_packs"])]
    swapped_bytes = sum(s.nbytes for s in saved_info if s.swapped)
    plan = SwapPlan(
        graph=g, rewritten=out, report=rep, n_packs=meta["n_packs"],
        pack_saved=[si if (si >= 0 and pack_is_swapped[k]) else -1 for k, si in enumerate(pack_saved)],
        saved=saved_info, groups=groups, pack_group=pack_group, triggers=triggers,
        bwd_start_groups=bwd_start, eager_groups=eager,
        swapped_bytes_per_step=swapped_bytes,
        saved_bytes_per_step=sum(s.nbytes for s in saved_info),
        capture_batch=capture_batch, rewrite_seconds=dt,
        fwd_groups=[g.gid for g in fwd_groups], fwd_triggers=fwd_triggers)
    _ = F
    return plan


def _forward_group(out: CompGraph, meta: dict, node: int, orig: int, si, fwd_cons, ctrl, gid):
    """The forward side of one branch swap-in node, or None when it stays an
    identity on the device (too small, or its ranks cannot be tracked)."""
    F = meta["F"]
    t = out.tensor_by_id[orig]
    if not meta.get("fwd_ranks_ok") or t.producer not in F or t.size_bytes < meta.get("min_swap_bytes", 0):
        return None
    prod = F[t.producer]
    # the device copy must stay until the forward readers the rewrite left in place have run
    keep = [F[e.dst] for e in out.consumer_edges(orig) if e.action is EdgeAction.READ and e.dst in F]
    release = max([prod] + keep)
    if ctrl is None:
        kind, trig = "eager", None
    elif ctrl in F:
        kind, trig = "forward", F[ctrl]
    else:
        return None
    return SwapGroup(gid, -1 if si is None else si, [], trig, kind, node, fwd_consumers=tuple(fwd_cons),
                     tensor=orig, producer_rank=prod, release_rank=release, nbytes=t.size_bytes)


def _issuer(issue, gids):
    def hook(grad_inputs, grad_outputs):
        for gid in gids:
            issue(gid)
        return None
    return hook


def _clocker(ctx, out, rank):
    def hook(grad_inputs, grad_outputs):
        out[rank] = ctx.plan_clock()
        return None
    return hook


def retarget(plan: SwapPlan, moves: dict) -> SwapPlan:
    """``plan`` with the swap-ins in ``moves`` ({gid: node rank}) fired by other
    backward nodes; each node issues its swap-ins in their original order."""
    from dataclasses import replace
    groups = [replace(g, trigger=moves[g.gid]) if g.gid in moves else g for g in plan.groups]
    triggers: dict[int, list] = {}
    for r, gids in plan.triggers.items():   # a node's own swap-ins first, in their order
        kept = [gid for gid in gids if gid not in moves]
        if kept:
            triggers[r] = kept
    for gid, r in moves.items():            # then the moved ones, in ``moves`` order
        triggers.setdefault(r, []).append(gid)
    return replace(plan, groups=groups, triggers=triggers)


def plan_window_moves(live, node_clock: dict, issue: list, cands: dict, trigger: dict, limit: float) -> list:
    """The model step of ``LMS.tune_windows`` (host only).

    ``live``: bytes live per event of a recorded step (updated in place);
    ``node_clock``: {node rank: event clock when it finished}; ``issue``:
    [(clock, gid, bytes)] of the swap-ins; ``cands``: {gid: [candidate node
    ranks]}; ``trigger``: {gid: current node rank}.  Swap-ins in issue order
    each take the earliest candidate c2 < c1 with max(live[c2:c1]) + bytes <=
    limit that does not pass the previous swap-in's trigger.  Returns
    [(gid, c1, c2, bytes, rank)] in issue order."""
    out, prev = [], -1
    for c1, gid, nb in sorted(issue):
        best = None
        for r in cands.get(gid, ()):
            c2 = node_clock.get(r)
            if r == trigger.get(gid) or c2 is None or c2 >= c1 or c2 < prev:
                continue
            if best is not None and c2 >= best[1]:
                continue
            if live[c2:c1].max() + nb <= limit:
                best = (r, c2)
        if best is None:
            prev = max(prev, c1)
            continue
        r, c2 = best
        live[c2:c1] += nb
        out.append((gid, c1, c2, nb, r))
        prev = c2
    return out


class _ForwardSwaps(TorchFunctionMode):
    """Forward-side interception for branch swaps (swap_branches, rewriter.py:231).

    Saved-tensor hooks only see tensors autograd keeps for backward; a U-Net
    skip tensor is also held by the model's own Python references until its
    forward consumer (the concatenation) runs, so its device copy can only go
    away if the forward pass itself lets go of the memory.  Every torch call
    of the forward passes through here:

    * after the op that produces a swapped branch tensor (its autograd node's
      rank), the D2H starts (one swap-out per tensor, shared with the
      saved-tensor path when autograd also saves it — fuse_swap_outs,
      rewriter.py:294-334);
    * after the last forward op the rewrite left reading the device copy, the
      tensor's storage is resized to 0 bytes: the block returns to the pool
      once the D2H lands (lms_swap_out holds it) while every Python reference
      and saved alias stays valid;
    * after the control op's node (rewriter.py:455-477) the storage is
      re-allocated and the H2D issued; an op reading a freed storage first
      makes the compute stream wait for its swap-in (issuing it if its control
      op never ran).
    """

    def __init__(self, ex: "SwapExecutor", issue_saved):
        super().__init__()
        plan = ex.plan
        self.ex, self.ctx = ex, ex.ctx
        self.issue_saved = issue_saved   # (saved idx, tensor) -> handle, shared with the pack hook
        self.groups = [plan.groups[g] for g in plan.fwd_groups]
        self.by_prod, self.by_release, self.by_trigger = {}, {}, {}
        for g in self.groups:
            self.by_prod.setdefault(g.producer_rank, []).append(g)
            self.by_release.setdefault(g.release_rank, []).append(g)
            if g.trigger_kind == "forward":
                self.by_trigger.setdefault(g.trigger, []).append(g)
        self.ranks = set(self.by_prod) | set(self.by_release) | set(self.by_trigger)
        self.seq0 = None
        self.state = {}      # tensor id -> dict(t, h, phase, key)
        self.freed = {}      # storage key -> tensor id
        self.n_freed = 0

    def _post(self, r, t):
        ctx, st = self.ctx, self.state
        for g in self.by_prod.get(r, ()):
            if g.tensor in st:
                continue
            whole = (t.storage_offset() == 0 and t.is_contiguous()
                     and t.numel() * t.element_size() == t.untyped_storage().nbytes())
            if not whole:
                st[g.tensor] = {"phase": "kept"}
                continue
            h = self.issue_saved(g.saved, t)
            st[g.tensor] = {"t": t, "h": h, "phase": "out", "eager": g.trigger_kind == "eager"}
        for g in self.by_release.get(r, ()):
            x = st.get(g.tensor)
            if x is None or x["phase"] != "out" or x["eager"]:
                continue
            stor = x["t"].untyped_storage()
            x["nbytes"], x["key"] = stor.nbytes(), stor._cdata
            stor.resize_(0)     # the pool reuses the block once the D2H has landed
            x["phase"] = "freed"
            self.freed[x["key"]] = g.tensor
            self.n_freed += 1
        for g in self.by_trigger.get(r, ()):
            x = st.get(g.tensor)
            if x is None:
                continue
            if x["phase"] == "freed":
                self._swap_in(x)
            elif x["phase"] == "out":
                x["eager"] = True    # control op before the release point: keep it resident

    def _swap_in(self, x):
        x["t"].untyped_storage().resize_(x["nbytes"])
        self.ctx.swap_in(x["h"], dst=x["t"], trigger_stream=torch.cuda.current_stream())
        x["phase"] = "in"

    def __torch_function__(self, func, types, args=(), kwargs=None):
        kwargs = kwargs or {}
        if self.freed:
            for a in tree_flatten((args, kwargs))[0]:
                if isinstance(a, torch.Tensor) and a.layout == torch.strided:
                    tid = self.freed.get(a.untyped_storage()._cdata)
                    if tid is not None:
                        x = self.state[tid]
                        if x["phase"] == "freed":
                            self._swap_in(x)
                        self.ctx.wait(x["h"], torch.cuda.current_stream())
                        x["phase"] = "restored"
                        x["t"] = None     # the model's own references decide its lifetime again
                        del self.freed[x["key"]]
        out = func(*args, **kwargs)
        seen = set()
        for t in tree_flatten(out)[0]:
            if isinstance(t, torch.Tensor) and t.grad_fn is not None:
                seq = t.grad_fn._sequence_nr()
                if self.seq0 is None:
                    self.seq0 = seq
                r = seq - self.seq0
                if r in self.ranks and r not in seen:
                    seen.add(r)
                    self._post(r, t)
        return out

    def finish(self):
        """End of forward: anything still freed is restored (its consumer never ran)."""
        for tid in list(self.freed.values()):
            x = self.state[tid]
            if x["phase"] == "freed":
                self._swap_in(x)
            self.ctx.wait(x["h"], torch.cuda.current_stream())
            x["phase"] = "restored"
            x["t"] = None
        self.freed.clear()
        # tensors swapped out but never freed (no release point reached) are not pinned either
        for x in self.state.values():
            x.pop("t", None)


class _SwapRef:
    """What autograd keeps instead of a swapped tensor."""

    __slots__ = ("k",)

    def __init__(self, k):
        self.k = k


class SwapExecutor:
    """Runs training steps under a :class:`SwapPlan` on one device."""

    def __init__(self, ctx: rt.Context, plan: SwapPlan, codec: str | dict = "ce", zx_max_ratio: float | None = None):
        self.ctx = ctx
        self.plan = plan
        self.codec = codec
        self.zx_max_ratio = self.ZX_MAX_RATIO if zx_max_ratio is None else zx_max_ratio
        self.last_stats = {}
        self.handle_tensor: dict[int, int] = {}   # lms handle id -> captured graph tensor id (last step)
        # window probe (LMS.tune_windows): {"ranks": node ranks to clock} -> the run
        # fills "node_clock" {rank: plan clock when the node finished on the host}
        # and "issue" {gid: (plan clock at the swap-in, bytes)}
        self.probe: dict | None = None

    # The codecs move encoded bytes with SM kernels at ~51 GB/s where the copy
    # engine moves raw bytes at ~57 (profiles/r02), so an encoded transfer wins
    # once its stream is below ~0.9 of the tensor.  The capture step measured
    # each saved tensor's ZX ratio with the codec's own tile rules (ReLU outputs
    # ~0.46: zero masks, no sign bit; conv/BN outputs ~0.89: 4 exponent bits and
    # a sign bit instead of 8 bits).  ResNet-50 at 908: ZX on both kinds
    # 331 img/s, ZX on ReLU outputs only 321 (profiles/r02/README.md).
    ZX_MAX_RATIO = 0.92
    # ... but an encoded transfer is moved by SM kernels that stay resident for
    # the whole (link-bound) copy, next to the compute stream's kernels.  When
    # the step's swap traffic is short next to its compute, the link has time
    # to spare and those SM slots only slow the compute down: ResNet-50 at
    # 1.25x B0 (4.9 GB swapped): copy engine 754.8 img/s, ZX on ReLU outputs
    # 736.7, ZX on everything 623.1; at 4.7x B0 (55 GB): ZX on everything is
    # the fastest (profiles/r02/README.md).
    @staticmethod
    def zx_policy(link_s: float, compute_s: float) -> float:
        """ZX threshold for a step whose swaps take ``link_s`` on the copy engine and
        whose compute takes ``compute_s``: none while the link is not the bottleneck,
        only clearly compressible tensors (ReLU outputs) near balance, every tensor
        the codec shrinks once the link decides the step."""
        r = link_s / max(compute_s, 1e-9)
        if r < 0.6:
            return 0.0
        if r < 1.2:
            return 0.6
        return 0.92

    def _codec_for(self, si: int, t) -> str:
        if self.codec == "auto":
            return "zx" if self.plan.saved[si].zx_ratio <= self.zx_max_ratio else "ce"
        if isinstance(self.codec, str):
            return self.codec
        return self.codec.get(si, "ce")

    def run(self, forward_fn):
        """``forward_fn()`` runs forward and returns the loss; backward happens here."""
        plan, ctx = self.plan, self.ctx
        k_counter = [0]
        handles: dict[int, rt.SwapHandle] = {}     # saved idx -> host copy
        group_tensor: dict[int, torch.Tensor] = {}
        group_waited: dict[int, int] = {}
        group_left = {g.gid: len(g.packs) for g in plan.groups}
        issued: set[int] = set()
        stream_of = torch.cuda.current_stream
        probe = self.probe
        if probe is not None:
            probe["node_clock"], probe["issue"] = {}, {}

        def issue(gid):
            if gid in issued:
                return
            grp = plan.groups[gid]
            h = handles.get(grp.saved)
            if h is None:
                return  # its swap-out never happened (structure changed); unpack will fail loudly
            issued.add(gid)
            if probe is not None:
                probe["issue"][gid] = (ctx.plan_clock(), h.logical_bytes)
            group_tensor[gid] = ctx.swap_in(h, trigger_stream=stream_of())

        def pack(t):
            k = k_counter[0]
            k_counter[0] = k + 1
            si = plan.pack_saved[k] if k < plan.n_packs else -1
            if si < 0:
                # detached alias, not ``t``: an op output saved as itself would
                # form a tensor -> grad_fn -> saved -> tensor cycle that only a
                # completed backward breaks (a step that fails in forward would
                # leak its activations)
                return t.detach()
            h = handles.get(si)
            if h is not None and (h.shape != tuple(t.shape) or h.restore_strides != tuple(t.stride())):
                # a branch swap-out of another view of it: autograd's copy is its own
                old = handles.pop(si)
                handles[("fwd", old.id)] = old
                h = None
            if h is None:
                h = ctx.swap_out(t, self._codec_for(si, t), stream_of())
                handles[si] = h
                self.handle_tensor[h.id] = plan.saved[si].tid
                for gid in plan.eager_groups:
                    if plan.groups[gid].saved == si:
                        issue(gid)
            return _SwapRef(k)

        def unpack(obj):
            if not isinstance(obj, _SwapRef):
                return obj
            gid = plan.pack_group[obj.k]
            if gid not in issued:
                issue(gid)  # control op did not fire (e.g. pruned branch): fetch now
            t = group_tensor.get(gid)
            if t is None:
                # unpacked again after the group was released: fetch once more
                issued.discard(gid)
                issue(gid)
                t = group_tensor[gid]
            ctx.wait(handles[plan.groups[gid].saved], stream_of())
            group_left[gid] -= 1
            if group_left[gid] <= 0:
                group_tensor.pop(gid, None)  # the consumer node holds it until it finishes
            return t

        def issue_saved(si, t):
            """The swap-out of a branch tensor: the saved-tensor path's handle when
            autograd saves it too (same layout), else a new one."""
            h = handles.get(si) if si >= 0 else None
            if h is not None and h.shape == tuple(t.shape) and h.restore_strides == tuple(t.stride()):
                return h
            h = ctx.swap_out(t, self._codec_for(si, t) if si >= 0 else "ce", stream_of())
            key = si if si >= 0 and si not in handles else ("fwd", h.id)
            handles[key] = h
            return h

        fwd = _ForwardSwaps(self, issue_saved) if plan.fwd_groups else None
        self.forward_swaps = fwd
        hooks = []
        loss = None
        nvtx = torch.cuda.nvtx
        try:
            nvtx.range_push("lms:forward")
            with torch.autograd.graph.saved_tensors_hooks(pack, unpack):
                if fwd is None:
                    loss = forward_fn()
                else:
                    with fwd:
                        loss = forward_fn()
                    fwd.finish()
            nvtx.range_pop()
            if k_counter[0] != plan.n_packs:
                raise RuntimeError(f"step saved {k_counter[0]} tensors but the plan was captured with "
                                   f"{plan.n_packs}; re-capture the plan for this model/step")
            # hook the control ops of this step's graph
            if plan.triggers or probe is not None:
                ops = sorted((n for n in _walk(loss.grad_fn) if not _is_accumulate(n)),
                             key=lambda n: n._sequence_nr())
                seq0 = ops[0]._sequence_nr()
                for n in ops:
                    r = n._sequence_nr() - seq0
                    if probe is not None and r in probe["ranks"]:
                        hooks.append(n.register_hook(_clocker(ctx, probe["node_clock"], r)))
                    gids = plan.triggers.get(r)
                    if gids:
                        hooks.append(n.register_hook(_issuer(issue, gids)))
            for gid in plan.bwd_start_groups:
                issue(gid)
            nvtx.range_push("lms:backward")
            loss.backward()
            nvtx.range_pop()
        except BaseException:
            # a failed step (e.g. the budget is too small) must not pin the
            # graph, the swapped-in tensors or the host copies: the exception's
            # traceback keeps this frame alive
            loss = None
            raise
        finally:
            for hk in hooks:
                hk.remove()
            hooks.clear()
            group_tensor.clear()
            if fwd is not None:
                fwd.state.clear()
            for h in handles.values():
                ctx.release(h)
            handles.clear()
        return loss


def _snapshot_training_state(module: torch.nn.Module, optimizer) -> dict:
    """Host copies of a module's parameters and buffers and of its optimizer's
    per-parameter state (restored by ``_restore_training_state``)."""
    with torch.no_grad():
        return {"module": [t.detach().to("cpu", copy=True) for t in (*module.parameters(), *module.buffers())],
                "opt": {p: {k: ((v.detach().to("cpu", copy=True), v.device) if torch.is_tensor(v) else (v, None))
                            for k, v in st.items()}
                        for p, st in optimizer.state.items()}}


def _restore_training_state(module: torch.nn.Module, optimizer, saved: dict) -> None:
    with torch.no_grad():
        for t, v in zip((*module.parameters(), *module.buffers()), saved["module"]):
            t.copy_(v)
        for p in list(optimizer.state):
            if p not in saved["opt"]:
                del optimizer.state[p]
        for p, st in saved["opt"].items():
            cur = optimizer.state[p]
            for k, (v, dev) in st.items():
                c = cur.get(k)
                if dev is not None and torch.is_tensor(c) and c.shape == v.shape and c.device == dev:
                    c.copy_(v)
                else:
                    cur[k] = v.to(dev) if dev is not None else v
    optimizer.zero_grad(set_to_none=True)


class LMS:
    """TFLMS for a PyTorch training step: capture once, rewrite, then train with swapping.

    ``LMS(model, loss_fn, optimizer, RewriteConfig(...), ctx)`` mirrors the
    paper's usage (``LMS(...).run(graph)``, PAPER §5): the rewrite knobs are
    exactly the reference's ``RewriteConfig``.
    """

    def __init__(self, model, loss_fn, optimizer, cfg: RewriteConfig, ctx: rt.Context,
                 codec="auto", min_swap_bytes: int = 1 << 16, static_plan: bool = True,
                 far_cfg: RewriteConfig | None = None, far_max_fraction: float = 0.0):
        self.model, self.loss_fn, self.optimizer = model, loss_fn, optimizer
        # static step plan (include/lms.h): step 0 after a (re)plan runs on the
        # dynamic pool, step 1 is recorded and placed, later steps replay it
        self.static_plan = static_plan
        self.far_cfg, self.far_max_fraction = far_cfg, far_max_fraction
        self._plan_step = 0
        self._plan_misses = 0
        self.plan_note = None
        self.cfg = cfg
        self.ctx = ctx
        self.codec = codec
        self.min_swap_bytes = min_swap_bytes
        self.plan: SwapPlan | None = None
        self.graph = None
        self.meta = None
        self._exec = None

    def capture(self, x, y):
        """Trace one step at (x, y) — no optimizer update — and build the swap plan."""
        self.optimizer.zero_grad(set_to_none=True)
        persistent = list(self.model.parameters()) + list(self.model.buffers()) + [x, y]
        # the traced step is not a training step: module buffers it updates
        # (BatchNorm running statistics, num_batches_tracked) are put back
        kept = [(b, b.detach().clone()) for b in self.model.buffers()]
        self.graph, self.meta = capture_graph(lambda: self.loss_fn(self.model(x), y), self.min_swap_bytes,
                                              persistent)
        with torch.no_grad():
            for b, v in kept:
                b.copy_(v)
        del kept
        self.optimizer.zero_grad(set_to_none=True)
        self.replan(self.cfg)
        return self.plan

    def replan(self, cfg: RewriteConfig):
        """Re-run the rewrite with new knobs on the captured graph (no re-trace)."""
        self._drop_step_plan()
        self.cfg = cfg
        self.plan = build_plan(self.graph, self.meta, cfg, 0, self.far_cfg, self.far_max_fraction)
        self._exec = SwapExecutor(self.ctx, self.plan, self.codec, self._zx_threshold(self.plan))
        return self.plan

    link_context = None   # (copy-engine GB/s, compute s per step, capture bytes -> step bytes)

    def set_link_context(self, link_gbs: float, compute_s: float, bytes_scale: float):
        """Let ``codec="auto"`` weigh each plan's swap traffic against the step's
        compute (``SwapExecutor.zx_policy``)."""
        self.link_context = (link_gbs, compute_s, bytes_scale)
        if self.plan is not None:
            self._exec.zx_max_ratio = self._zx_threshold(self.plan)

    def _zx_threshold(self, plan) -> float:
        if self.link_context is None:
            return SwapExecutor.ZX_MAX_RATIO
        gbs, compute_s, scale = self.link_context
        return SwapExecutor.zx_policy(plan.swapped_bytes_per_step * scale / (gbs * 1e9), compute_s)

    PLAN_ATTEMPTS = 3
    # replay steps that re-place the plan with the lifetimes they observe (the
    # recorded step ran on the dynamic pool and is slower than a replay)
    REFINE_STEPS = (2,)
    TRIM_ZOMBIES = 256   # 64 MiB pages: 16 GiB of stale VA

    def autotune(self, x, y, lbs=(1, 2, 3, 5, 8), steps: int = 3):
        """Pick the control-op window empirically (the paper leaves the lb/ub
        heuristic open): for each lb, run ``steps`` swapped steps
        at this batch (the last one timed with CUDA events); keep the fastest lb
        that fits the budget.  Returns ``{lb: ms per step or None (OOM)}``; the
        model's parameters move by ``len(lbs) * steps`` optimizer steps."""
        from dataclasses import replace
        base = self.cfg
        timings = {}
        for lb in lbs:
            self.replan(replace(base, lb=lb, ub=max(base.ub, lb)))
            try:
                for _ in range(max(1, steps - 1)):
                    self.step(x, y)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                self.step(x, y)
                e1.record()
                torch.cuda.synchronize()
                timings[lb] = e0.elapsed_time(e1)
            except (torch.OutOfMemoryError, rt.LmsOutOfMemoryError):
                timings[lb] = None
                self.optimizer.zero_grad(set_to_none=True)
                torch.cuda.synchronize()
                self.ctx.synchronize()
        fits = {lb: ms for lb, ms in timings.items() if ms is not None}
        best = min(fits, key=fits.get) if fits else base.lb
        self.replan(replace(base, lb=best, ub=max(base.ub, best)))
        return timings

    def tune_windows(self, x, y, lbs=(2, 3, 4, 5, 6, 8, 12, 16, 24, 32, 48, 64, 96), margin: float = 0.005,
                     require_faster: bool = True, steps: int = 5, agree=None, max_trials: int = 4,
                     deadline_s: float | None = None) -> dict:
        """Memory-aware control-op windows, one per swap-in (an extension: the
        paper leaves choosing lb open).  Every candidate control
        op comes from the reference's own strategy run with a wider window
        (``rewrite`` at each lb in ``lbs``, same swap nodes), so each chosen edge
        is one the rewrite itself could emit.

        One recorded step under the current plan gives the device pool's live
        bytes on its event clock (``lms_plan_items``) and, for every candidate
        node, the clock at which it finished on the host (``lms_plan_clock``).
        Moving a swap-in from clock c1 to an earlier node at c2 keeps its
        destination live over [c2, c1); swap-ins are visited in issue order and
        each takes the earliest candidate that keeps the live bytes under the
        pool's room (less ``margin``) and does not pass the previous swap-in's
        trigger (the H2D channel stays in consumer order).  The longest prefix
        of those moves whose placement the pool's solver fits is then tried
        for real: re-targeted (``retarget``), re-recorded and one replayed step
        timed against the untouched plan; the set shrinks by a third until a replay
        fits and is faster, or dropped (when the untouched plan's own recording
        does not fit, the full set gets one try).  The model parameters move by the
        probe and trial steps (like ``autotune``).  Returns a summary dict;
        ``{}`` changes nothing (no room, or no static plan to measure).

        Each replay times ``steps`` steps (median and spread reported).  The
        winning trial's recorded placement is kept: the next steps replay the
        very placement that was timed.  Under DDP every rank must take the same
        number of steps: ``agree(value, op)`` (an all-reduce, op "max"/"min")
        makes every timing- and memory-dependent decision common to all ranks
        (slowest rank's times, any rank's failure).

        Under DDP (``agree`` given and the model a ``DistributedDataParallel``)
        tuning is side-effect free and collective-free inside a step: trials run
        the wrapped module's local replica (no gradient all-reduce), so a rank
        that hits the budget mid-step strands no peer in a collective; it keeps
        joining every ``agree`` with a failure vote instead.  The weights,
        buffers and optimizer state are restored at the end, so the replicas
        stay identical.

        At most ``max_trials`` shrinking trials are timed, and none is started
        past ``deadline_s`` seconds from the call (the slowest rank's clock)."""
        with self._local_replica(agree):
            return self._tune_windows(x, y, lbs, margin, require_faster, steps, agree, max_trials, deadline_s)

    @contextlib.contextmanager
    def _local_replica(self, agree):
        """Under DDP with ``agree``: run the wrapped module alone (no collective
        inside a step) and put weights, buffers and optimizer state back after.
        The step plan recorded on the local replica is dropped on the way out:
        the wrapped steps allocate differently (a bucket rebuild on a fresh
        wrapper's second step takes ~the gradients' bytes before the old
        buckets go), so they record their own; the swap plan and its tuned
        windows stay."""
        ddp = self.model if isinstance(self.model, torch.nn.parallel.DistributedDataParallel) else None
        if agree is None or ddp is None:
            yield
            return
        saved = _snapshot_training_state(ddp.module, self.optimizer)
        self.model = ddp.module
        try:
            yield
        finally:
            self.model = ddp
            _restore_training_state(ddp.module, self.optimizer, saved)
            self._drop_step_plan()

    def time_replay(self, x, y, steps: int = 5, agree=None):
        """Record the current plan once more and time ``steps`` replayed steps
        (``_timed_replay``); under DDP on the local replica like ``tune_windows``.
        The next steps replay the placement that was timed."""
        with self._local_replica(agree):
            return self._timed_replay(x, y, steps, agree)

    def _tune_windows(self, x, y, lbs, margin, require_faster, steps, agree, max_trials=4, deadline_s=None) -> dict:
        t_call = time.perf_counter()
        from dataclasses import replace
        import numpy as np
        if not self.static_plan or self.plan is None:
            return {}
        base = self.cfg
        B = self.meta["B"]
        node_of = {g.node: g.gid for g in self.plan.groups if g.trigger_kind == "backward"}
        cands: dict[int, list] = {gid: [] for gid in node_of.values()}
        for lb in lbs:
            out, _ = rewrite(self.graph, replace(base, lb=lb, ub=max(base.ub, lb)))
            for e in out.edges:
                if e.action is EdgeAction.CONTROL and e.dst in node_of and e.src in B:
                    cands[node_of[e.dst]].append(B[e.src])
        ranks = {r for v in cands.values() for r in v}
        if not ranks:
            return {}
        # step 0 of the plan runs dynamic; step 1 records with the probe on
        def common(v, op):
            return v if agree is None else agree(v, op)

        # the recorded step the moves are modelled on varies with transfer timing:
        # when none of the modelled moves fits its room, record once more
        for attempt in range(2):
            self._drop_step_plan()
            probe = {"ranks": ranks}
            ok = True
            try:
                while self._plan_step != 1:
                    self.step(x, y)
                self._exec.probe = probe
                try:
                    self.step(x, y)
                finally:
                    self._exec.probe = None
                torch.cuda.synchronize()
            except (torch.OutOfMemoryError, rt.LmsOutOfMemoryError):
                if agree is None:
                    raise
                ok = False      # vote failure below; no collective was left half-done
                self._after_oom()
            if common(1.0 if ok and self.plan_note == "region" else 0.0, "min") < 0.5:
                self._drop_step_plan()
                return {}
            info = self.ctx.plan_info()
            items = self.ctx.plan_items()
            T = max((max(a, b, c) for _, a, b, c in items), default=0) + 2
            live = np.zeros(T, dtype=np.float64)
            for size, a, b, c in items:
                if b >= 0:
                    live[a:b] += size
            # the next recording's room: the pages not live once this plan's region
            # is returned, less the page the pool keeps for unplanned allocations
            limit = info["room_bytes"] * (1.0 - margin) - (64 << 20)
            start_peak = float(live.max()) if T else 0.0
            node_clock = probe["node_clock"]
            issue = sorted(((c, gid, nb) for gid, (c, nb) in probe["issue"].items() if gid in cands))
            moved = plan_window_moves(live, node_clock, issue, cands,
                                      {g.gid: g.trigger for g in self.plan.groups}, limit)
            # the live bytes bound the placement from below only: keep the longest
            # prefix of the moves (in issue order) whose recorded step, with those
            # destinations allocated at their new clocks, still places inside the
            # room (the pool's own solver, lms_plan_solve)
            sizes = [it[0] for it in items]
            t0 = [it[1] for it in items]
            t1 = [it[2] for it in items]
            item_at = {a: i for i, a in enumerate(t0)}
            # a move is modelled only if its destination is the allocation made at
            # its issue clock (same bytes up to the pool's rounding)
            moved = [m for m in moved if m[1] in item_at and 0 <= sizes[item_at[m[1]]] - m[3] < (4 << 20)]

            def region_with(k):
                tk = list(t0)
                for gid, c1, c2, nb, _ in moved[:k]:
                    tk[item_at[c1]] = c2
                return rt.plan_solve(sizes, tk, t1)[1]

            keep = len(moved)
            if moved and region_with(keep) > limit:
                lo, hi = 0, keep      # lo fits (the recorded plan), hi does not
                while hi - lo > 1:
                    mid = (lo + hi) // 2
                    if region_with(mid) <= limit:
                        lo = mid
                    else:
                        hi = mid
                keep = lo
            # each rank models its own recorded step; the trial schedule is common
            keep = int(common(float(keep), "min"))
            if keep > 0 or attempt == 1 or common(float(len(moved)), "max") == 0:
                break
        # the model predicts; replayed steps decide: re-record with the moves,
        # keep them if the placement fits at the physical-release lifetimes
        # (alpha 1: no block reused before its swap-out copy landed) and the
        # replayed steps are faster than the untouched plan's; else shrink the set
        orig = self.plan
        base = self._timed_replay(x, y, steps, agree)
        base_ms = base["ms"] if base else None
        trials, spreads = {}, {"base": base["spread"] if base else None}
        chosen = 0
        while keep > 0 and len(trials) < max_trials:
            if deadline_s is not None and common(time.perf_counter() - t_call, "max") > deadline_s:
                break
            self._set_plan(retarget(orig, {m[0]: m[4] for m in moved[:keep]}))
            r = self._timed_replay(x, y, steps, agree)
            trials[keep] = r["ms"] if r else None
            spreads[keep] = r["spread"] if r else None
            if r is not None and (base_ms is None or r["ms"] < base_ms or not require_faster):
                chosen = keep
                break
            if base_ms is None:
                break       # the untouched plan's recording did not fit either: one try with every move
            keep = keep * 2 // 3
        if not chosen:
            # the untouched plan won: replay it again so its recorded placement is the one kept
            self._set_plan(orig)
            again = self._timed_replay(x, y, steps, agree) if base_ms is not None else None
            final = again["ms"] if again else None
        else:
            final = trials[chosen]   # the winner's recording is the live plan: kept as is
        return {"moved": chosen, "of": len(issue), "modelled": len(moved),
                "moved_bytes": sum(m[3] for m in moved[:chosen]),
                "base_ms": base_ms, "trials": trials, "spread_ms": spreads, "final_ms": final,
                "steps_per_trial": steps, "peak_before": start_peak,
                "limit": limit, "lower_bound": info["lower_bound_bytes"]}

    def plan_by_model(self, x, y, cfgs, batch: int, link, budget_bytes: int, capture_batch: int = 4):
        """Rank candidate ``RewriteConfig``s by the calibrated model (calibrate.py):
        one plain step at (x, y) — a batch that fits without swapping — is timed
        per captured node and gives the fixed (non-activation) bytes; costs and
        tensor sizes are scaled to ``batch``; each config's rewrite of the
        captured graph is predicted.  Returns ``[(cfg, prediction, fits)]``,
        fitting configs fastest first.  The model's parameters move by one
        optimizer step (like ``autotune``)."""
        from . import calibrate as cal
        b = x.shape[0]
        torch.cuda.synchronize()
        self.ctx.reset_peaks()
        live0 = self.ctx.stats()["device_in_use"]
        costs = cal.node_costs(self.model, self.loss_fn, x, y, self.meta, self.optimizer)
        plain_peak = self.ctx.stats()["device_peak"] - live0
        g_b = cal.calibrated_graph(self.graph, costs, b / capture_batch, 1.0, costs["_optimizer_total"], self.meta)
        fixed = plain_peak - cal.predict(g_b, link)["peak_device_bytes"]
        g_t = cal.calibrated_graph(self.graph, costs, batch / capture_batch, batch / b, costs["_optimizer_total"],
                                   self.meta)
        self.model_costs, self.model_fixed_bytes, self.model_graph = costs, fixed, g_t
        self.model_room = budget_bytes - fixed
        return cal.plan_ranking(g_t, cfgs, link, budget_bytes - fixed)

    def link_model(self, link_gbs: dict, zc_efficiency: float = 0.9):
        """A ``calibrate.LinkModel`` from measured copy-engine rates (GB/s, bench's
        ``measure_host_link``) and the capture step's per-tensor ZX ratios."""
        from .calibrate import LinkModel
        wire = {self.meta["saved_tensor_id"][s.tid]: s.zx_ratio for s in self.meta["saved"]
                if s.tid in self.meta["saved_tensor_id"]}
        return LinkModel(d2h_ce=link_gbs["d2h"] * 1e9, h2d_ce=link_gbs["h2d"] * 1e9,
                         d2h_zc=zc_efficiency * link_gbs["d2h"] * 1e9, h2d_zc=zc_efficiency * link_gbs["h2d"] * 1e9,
                         wire_ratio=wire, zx_max_ratio=self._exec.zx_max_ratio if self._exec else
                         SwapExecutor.ZX_MAX_RATIO)

    def _set_plan(self, plan: SwapPlan):
        self.plan = plan
        self._exec = SwapExecutor(self.ctx, plan, self.codec, self._zx_threshold(plan))
        self._drop_step_plan()

    def _timed_replay(self, x, y, steps: int = 5, agree=None):
        """Re-record the current plan (dynamic, recorded and first replayed step) and
        time ``steps`` replayed ones.  Returns {"ms": median ms per step, "spread":
        (min, max)} or None if the placement does not fit at physical-release
        lifetimes or a step hits the budget.  The step count is fixed, so DDP ranks
        stay in step; ``agree`` makes the outcome common (slowest rank, any failure)."""
        self._drop_step_plan()
        failed = False

        def run_step():
            # under ``agree`` a rank that hits the budget stops stepping but keeps
            # voting, so every rank makes the same sequence of all-reduces
            nonlocal failed
            if failed:
                return
            try:
                self.step(x, y)
            except (torch.OutOfMemoryError, rt.LmsOutOfMemoryError):
                if agree is None:
                    raise
                failed = True
                self._after_oom()

        per = None
        try:
            # dynamic step, recorded step, first replay; a recording whose placement
            # did not fit is retried (at most 6 setup steps; under DDP the ranks
            # agree on when every one of them is done)
            for _ in range(6):
                done = failed or self._plan_step >= 3 or self.plan_note == "no-fit"
                if agree is not None:
                    done = agree(1.0 if done else 0.0, "min") > 0.5
                if done:
                    break
                run_step()
            fits = not failed and self.plan_note == "region" and self.ctx.plan_info()["alpha"] >= 1.0
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
            torch.cuda.synchronize()
            evs[0].record()
            for k in range(steps):
                run_step()
                evs[k + 1].record()
            torch.cuda.synchronize()
            per = sorted(evs[k].elapsed_time(evs[k + 1]) for k in range(steps)) if fits and not failed else None
        except (torch.OutOfMemoryError, rt.LmsOutOfMemoryError):
            self._after_oom()       # agree is None here: run_step re-raised
        if agree is not None:
            if agree(0.0 if per is None else 1.0, "min") < 0.5:
                return None
            per = [agree(v, "max") for v in per]
        if per is None:
            return None
        return {"ms": per[len(per) // 2], "spread": (per[0], per[-1])}

    def trace_events(self):
        """The last steps' measured transfers as the reference's ``TraceEvent``s
        (``sim.py:74-81``): ``xfer_start``/``xfer_finish`` per swap, time in
        seconds from the context epoch, tensor = the captured graph's tensor id,
        device = where the bytes land.  ``write_trace_csv`` writes them in the
        reference's CSV schema, so measured and simulated timelines diff."""
        from .report import TraceEvent
        ev = []
        tids = self._exec.handle_tensor if self._exec else {}
        for r in self.ctx.trace():
            tid = self.meta["saved_tensor_id"].get(tids.get(r["handle_id"])) if self.meta else None
            where = "host" if r["direction"] == 0 else f"acc:{self.ctx.device}"
            ev.append(TraceEvent(r["start_ms"] * 1e-3, "xfer_start", None, tid, r["wire_bytes"], where))
            ev.append(TraceEvent(r["end_ms"] * 1e-3, "xfer_finish", None, tid, r["wire_bytes"], where))
        ev.sort(key=lambda e: e.time)
        return ev

    def _after_oom(self):
        """Clean up after a step that hit the budget: no gradients, idle streams,
        no half-recorded plan."""
        self.optimizer.zero_grad(set_to_none=True)
        torch.cuda.synchronize()
        self.ctx.synchronize()
        self._drop_step_plan()

    def _drop_step_plan(self):
        if self._plan_step >= 2 or self.plan_note == "region":
            torch.cuda.synchronize()
            self.ctx.plan_reset()
        self._plan_step = 0
        self._plan_misses = 0
        self.plan_note = None

    def step(self, x, y):
        """One swapped training step; returns the loss tensor (on device)."""
        mode = rt.PLAN_OFF
        if self.static_plan and self.plan_note != "no-fit":
            mode = (rt.PLAN_RECORD if self._plan_step == 1
                    else rt.PLAN_REFINE if self._plan_step in self.REFINE_STEPS and self.plan_note == "region"
                    else rt.PLAN_REPLAY if self._plan_step >= 2 else rt.PLAN_OFF)
        if mode == rt.PLAN_RECORD:
            torch.cuda.synchronize()
            try:
                self.ctx.plan_reset()   # a plan left over from a failed step
            except rt.LmsError:
                # blocks of the failed step's plan are still referenced: run this
                # step on the dynamic pool and record the next one
                mode = rt.PLAN_OFF
                self._plan_step = 0
        if mode != rt.PLAN_OFF:
            self.ctx.plan_begin(mode)
        try:
            self.optimizer.zero_grad(set_to_none=True)
            loss = self._exec.run(lambda: self.loss_fn(self.model(x), y))
            self.optimizer.step()
        except BaseException:
            if mode != rt.PLAN_OFF:
                self.ctx.plan_begin(rt.PLAN_OFF)   # abandon the step's recording/replay
            self.optimizer.zero_grad(set_to_none=True)
            try:
                self._drop_step_plan()
            except rt.LmsError:
                self._plan_step = 0
            raise
        if mode != rt.PLAN_OFF:
            try:
                self.ctx.plan_end()
                if mode == rt.PLAN_RECORD:
                    self.plan_note = "region"
            except rt.LmsOutOfMemoryError:
                # the placement does not fit next to the live set: record again
                # (lifetimes vary with transfer timing), then stay dynamic
                self._plan_misses += 1
                if self._plan_misses < self.PLAN_ATTEMPTS:
                    self._plan_step = 0
                else:
                    self.plan_note = "no-fit"
        self._plan_step += 1
        # page moves leave stale VA aliases; unmapping them drains the device,
        # so it happens here, between steps, once they add up to ~1/4 of the
        # pool's reserved VA (a step in replay makes none)
        self.ctx.trim(self.TRIM_ZOMBIES)
        return loss
