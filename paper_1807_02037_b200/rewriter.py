"""The swap rewrite: insert swap-out/swap-in pairs and their control edges.

Drop-in for ``swapgraph/rewriter.py``: same ``RewriteConfig`` knobs (paper
Table 2), same ``RewriteReport`` schema, same pass functions and the same
``rewrite(g, cfg) -> (graph, report)`` entry point.  Output graphs are
byte-identical under ``dumps`` (ids, names, control edges, skip notes);
``tests/test_rewrite_parity.py`` pins this against golden vectors produced
by the reference itself.

The implementation is batch-oriented instead of edit-by-edit:

* all swap pairs are inserted in one sweep over plain lists (the reference
  rebuilds the whole ``CompGraph`` per insert, ``rewriter.py:241-277``);
* the control stage uses one :class:`~.control.CtrlIndex` over the query
  graph (ancestor bitsets, per-level op lists) and a bitset descendant
  closure for the cycle check, instead of O(V+E) searches per swap-in
  (``rewriter.py:455-477``, ``control.py:158-169``).

Reference anchors: ``RewriteConfig`` rewriter.py:41-80, ``RewriteReport``
:83-100, ``scope_matches`` :103-105, ``resolve_phases`` :116-139,
``_starting_nodes`` :142-157, ``select_candidates`` :160-211,
``_classify_edge`` :214-238, ``insert_swap_pair`` :241-277,
``fuse_swap_outs`` :294-334, ``fuse_swap_ins`` :337-396, ``rewrite``
:407-489.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass, field
from typing import Any

from . import control as ctrl
from .graph import (
    HOST,
    CompGraph,
    EdgeAction,
    EdgeRec,
    NodeKind,
    OpNode,
    Phase,
    SWAP_KINDS,
    TensorSpec,
    is_accelerator,
    topo_order,
    validate,
)

log = logging.getLogger("swapgraph")

_READ = EdgeAction.READ
_UPDATE = EdgeAction.UPDATE
_CONTROL = EdgeAction.CONTROL


class RewriteError(ValueError):
    """A pipeline stage failed; the message starts with ``stage '<name>':``."""


@dataclass(frozen=True)
class RewriteConfig:
    """Paper Table 2 knobs (defaults: lb=1, ub=10000, chain_rule, fusion off).

    ``optimizer_scopes`` phases untagged nodes; ``n_tensors`` caps distinct
    swapped tensors (-1 = all); ``lb``/``ub`` bound the control-op search;
    ``fuse_swapins``/``swapin_fuse_distance`` merge nearby swap-ins;
    ``swap_branches``/``branch_threshold`` also swap long forward->forward
    edges.
    """

    optimizer_scopes: frozenset[str] = frozenset()
    starting_scope: str | None = None
    starting_op_names: frozenset[str] = frozenset()
    excl_scopes: frozenset[str] = frozenset()
    incl_scopes: frozenset[str] = frozenset()
    excl_types: frozenset[str] = frozenset()
    incl_types: frozenset[str] = frozenset()
    n_tensors: int = -1
    lb: int = 1
    ub: int = 10000
    ctrld_strategy: str = "chain_rule"
    fuse_swapins: bool = False
    swapin_fuse_distance: int = 1
    swap_branches: bool = False
    branch_threshold: int = 0

    def __post_init__(self):
        checks = (
            (self.lb < 1, "lb must be positive"),
            (self.ub < self.lb, "ub must be >= lb"),
            (self.n_tensors < -1, "n_tensors must be -1 (all) or >= 0"),
            (self.ctrld_strategy not in ("chain_rule", "direct_order"),
             f"unknown ctrld_strategy {self.ctrld_strategy!r}"),
            (self.swapin_fuse_distance < 0, "swapin_fuse_distance must be >= 0"),
            (self.branch_threshold < 0, "branch_threshold must be >= 0"),
        )
        for bad, msg in checks:
            if bad:
                raise ValueError(msg)


@dataclass
class RewriteReport:
    tensors_swapped: int = 0
    swap_outs_added: int = 0
    swap_ins_added: int = 0
    control_edges_added: int = 0
    edges_rewritten: list[tuple[int, int, int]] = field(default_factory=list)
    skipped: list[dict[str, Any]] = field(default_factory=list)

    def to_dict(self) -> dict[str, Any]:
        d = {k: getattr(self, k) for k in
             ("tensors_swapped", "swap_outs_added", "swap_ins_added", "control_edges_added")}
        d["edges_rewritten"] = [list(e) for e in self.edges_rewritten]
        d["skipped"] = self.skipped
        return d


# -- filters ------------------------------------------------------------------

def scope_matches(scope: str, pattern: str) -> bool:
    """Component-prefix match: ``a/b`` matches ``a`` and ``a/b`` but not ``a/bc``."""
    if scope == pattern:
        return True
    return scope.startswith(pattern) and scope[len(pattern):len(pattern) + 1] == "/"


def _any_scope(scope: str, patterns) -> bool:
    for p in patterns:
        if scope_matches(scope, p):
            return True
    return False


def _type_hit(node: OpNode, tags) -> bool:
    return node.kind.value in tags or node.name in tags


# -- phases -------------------------------------------------------------------

def resolve_phases(g: CompGraph, optimizer_scopes) -> CompGraph:
    """Tag UNKNOWN-phase compute ops from optimizer scope membership.

    Inside an optimizer scope: UPDATE if the op writes a variable, else
    BACKWARD; elsewhere FORWARD.  Tagged, parameterized and swap nodes keep
    their phase.  No scopes: ``g`` is returned as is (rewriter.py:116-139).
    """
    if not optimizer_scopes:
        return g
    retagged = []
    changed = False
    for n in g.nodes:
        if n.parameterized or n.phase is not Phase.UNKNOWN or n.kind in SWAP_KINDS:
            retagged.append(n)
            continue
        if _any_scope(n.scope, optimizer_scopes):
            writes = any(e.action is _UPDATE for e in g.out_edges(n.id))
            ph = Phase.UPDATE if writes else Phase.BACKWARD
        else:
            ph = Phase.FORWARD
        retagged.append(OpNode(n.id, n.name, n.scope, n.kind, n.parameterized, ph,
                               n.device, n.cost_hint))
        changed = True
    if not changed:
        return CompGraph(g.nodes, g.edges, g.tensors)
    return CompGraph(retagged, g.edges, g.tensors)


def _phases_resolvable(g: CompGraph, cfg: RewriteConfig) -> bool:
    return bool(cfg.optimizer_scopes) or any(
        n.phase is not Phase.UNKNOWN for n in g.nodes if not n.parameterized)


# -- selection ----------------------------------------------------------------

def _starting_nodes(g: CompGraph, cfg: RewriteConfig) -> list[int]:
    if cfg.starting_scope is None and not cfg.starting_op_names:
        return [n.id for n in g.nodes if n.parameterized]  # nodes are id-sorted
    picked: set[int] = set()
    if cfg.starting_scope is not None:
        hit = {n.id for n in g.nodes if scope_matches(n.scope, cfg.starting_scope)}
        if not hit:
            raise ValueError(f"starting scope {cfg.starting_scope!r} matches no node")
        picked.update(hit)
    if cfg.starting_op_names:
        names = {n.name for n in g.nodes}
        missing = cfg.starting_op_names - names
        if missing:
            raise ValueError(f"starting op names match no node: {sorted(missing)}")
        picked.update(n.id for n in g.nodes if n.name in cfg.starting_op_names)
    return sorted(picked)


def _classify_edge(g: CompGraph, order: dict[int, int], cfg: RewriteConfig, e: EdgeRec) -> str:
    """'candidate', 'excluded' or 'no' for one read edge (rewriter.py:214-238)."""
    nbi = g.node_by_id
    src = nbi.get(e.src)
    dst = nbi.get(e.dst)
    if src is None or dst is None or e.tensor is None:
        return "no"
    if (src.parameterized or dst.parameterized
            or src.kind in SWAP_KINDS or dst.kind in SWAP_KINDS
            or not is_accelerator(src.device) or not is_accelerator(dst.device)):
        return "no"
    fwd = Phase.FORWARD
    hit = (
        (src.phase is fwd and dst.phase is Phase.BACKWARD)
        or (cfg.swap_branches and src.phase is fwd and dst.phase is fwd
            and order[e.dst] - order[e.src] > cfg.branch_threshold)
        or _any_scope(src.scope, cfg.incl_scopes)
        or _type_hit(src, cfg.incl_types)
    )
    if not hit:
        return "no"
    if _any_scope(src.scope, cfg.excl_scopes) or _type_hit(src, cfg.excl_types):
        return "excluded"
    return "candidate"


def _edge_visit_key(e: EdgeRec):
    return (e.dst, -1 if e.tensor is None else e.tensor)


def select_candidates(g: CompGraph, order: dict[int, int], cfg: RewriteConfig,
                      report: RewriteReport | None = None) -> list[tuple[EdgeRec, int]]:
    """(edge, tensor) pairs to rewrite, in breadth-first discovery order.

    BFS from the starting nodes (default: every parameterized node); each
    node's non-update out-edges are visited in (dst, tensor) order.  A tensor
    already kept keeps all its later edges even past the ``n_tensors`` cap;
    the cap only refuses new tensors (rewriter.py:160-211).
    """
    picked: list[tuple[EdgeRec, int]] = []
    kept: set[int] = set()
    cap = cfg.n_tensors
    queue = _starting_nodes(g, cfg)
    seen = set(queue)
    nbi = g.node_by_id
    pos = 0
    while pos < len(queue):
        nid = queue[pos]
        pos += 1
        outs = [e for e in g.out_edges(nid) if e.action is not _UPDATE]
        outs.sort(key=_edge_visit_key)
        for e in outs:
            if e.action is _READ:
                verdict = _classify_edge(g, order, cfg, e)
                if verdict == "candidate":
                    tid = e.tensor
                    if tid not in kept:
                        if 0 <= cap <= len(kept):
                            if report is not None:
                                report.skipped.append({"reason": "over n_tensors cap",
                                                       "tensor": tid, "edge": [e.src, e.dst]})
                            continue  # the dst is not enqueued from this edge
                        kept.add(tid)
                    picked.append((e, tid))
                elif verdict == "excluded" and report is not None:
                    report.skipped.append({"reason": "matched exclusion filter",
                                           "tensor": e.tensor, "edge": [e.src, e.dst]})
            if e.dst not in seen and e.dst in nbi:
                seen.add(e.dst)
                queue.append(e.dst)
    return picked


# -- insertion (paper Eq. 5) ------------------------------------------------------

def _swap_pair_records(t: TensorSpec, dst: int, so_id: int, so_tid: int):
    si_id, si_tid = so_id + 1, so_tid + 1
    so = OpNode(so_id, f"swap_out_{t.id}_{dst}", "swap", NodeKind.SWAP_OUT, False,
                Phase.UNKNOWN, HOST, 0.0)
    si = OpNode(si_id, f"swap_in_{t.id}_{dst}", "swap", NodeKind.SWAP_IN, False,
                Phase.UNKNOWN, HOST, 0.0)
    tensors = (TensorSpec(so_tid, so_id, t.size_bytes, t.dtype),
               TensorSpec(si_tid, si_id, t.size_bytes, t.dtype))
    return so, si, tensors


def insert_swap_pair(g: CompGraph, edge: EdgeRec) -> tuple[CompGraph, int, int]:
    """Replace read edge u->v (tensor t) with u->swap_out->swap_in->v.

    New node ids are max+1/max+2, new tensor ids likewise; both nodes are
    host-placed identities scoped ``swap`` (rewriter.py:241-277).
    """
    edges = list(g.edges)
    try:
        idx = edges.index(edge)
    except ValueError:
        raise ValueError(f"edge {edge} not present in graph") from None
    if edge.action is not _READ:
        raise ValueError(f"only read edges can be rewritten, got {edge.action.value}")
    src, dst = g.node_by_id[edge.src], g.node_by_id[edge.dst]
    if not (is_accelerator(src.device) and is_accelerator(dst.device)):
        raise ValueError(f"edge {edge.src} -> {edge.dst} is not between accelerator ops")
    t = g.tensor_by_id[edge.tensor]
    so_id = g.max_node_id() + 1
    so_tid = g.max_tensor_id() + 1
    so, si, new_t = _swap_pair_records(t, edge.dst, so_id, so_tid)
    del edges[idx]
    edges += (EdgeRec(edge.src, so_id, _READ, t.id),
              EdgeRec(so_id, so_id + 1, _READ, so_tid),
              EdgeRec(so_id + 1, edge.dst, _READ, so_tid + 1))
    return CompGraph(g.nodes + (so, si), edges, g.tensors + new_t), so_id, so_id + 1


# -- fusion -----------------------------------------------------------------------

def _only_read_input(g: CompGraph, nid: int) -> EdgeRec:
    reads = [e for e in g.in_edges(nid) if e.action is _READ]
    if len(reads) != 1:
        raise ValueError(f"swap node {nid} must have exactly one data input, has {len(reads)}")
    return reads[0]


def _only_output(g: CompGraph, nid: int) -> TensorSpec:
    outs = g.produced_tensors(nid)
    if len(outs) != 1:
        raise ValueError(f"swap node {nid} must produce exactly one tensor, has {len(outs)}")
    return outs[0]


def _merge_into(g: CompGraph, merged: dict[int, int]) -> CompGraph:
    """Drop every node in ``merged`` (victim -> survivor) and reroute its consumers."""
    if not merged:
        return g
    out_of = {v: _only_output(g, v).id for v in merged}
    reroute = {out_of[v]: (s, _only_output(g, s).id) for v, s in merged.items()}
    dead_t = set(reroute)
    edges = []
    for e in g.edges:
        if e.dst in merged:
            continue  # the victim's own input edge goes with it
        if e.src in merged:
            s, st = reroute[e.tensor]
            edges.append(EdgeRec(s, e.dst, e.action, st))
        else:
            edges.append(e)
    return CompGraph([n for n in g.nodes if n.id not in merged], edges,
                     [t for t in g.tensors if t.id not in dead_t])


def fuse_swap_outs(g: CompGraph) -> CompGraph:
    """One swap-out per (producer, tensor); lowest id survives (paper §4.2.2)."""
    by_source: dict[tuple[int, int], list[int]] = {}
    for n in g.nodes:
        if n.kind is NodeKind.SWAP_OUT:
            e = _only_read_input(g, n.id)
            by_source.setdefault((e.src, e.tensor), []).append(n.id)
    merged: dict[int, int] = {}
    for ids in by_source.values():
        if len(ids) > 1:
            keep = min(ids)
            for v in ids:
                if v != keep:
                    merged[v] = keep
    return _merge_into(g, merged)


def fuse_swap_ins(g: CompGraph, order: dict[int, int], distance_threshold: int) -> CompGraph:
    """Merge swap-ins of one swap-out whose consumers sit close (paper §4.2.3).

    Per swap-out, swap-ins are sorted by (earliest consumer order, id) and
    clustered greedily; a member joins while it is within
    ``distance_threshold`` of the cluster's first member.  The lowest id of
    each cluster survives and feeds all its consumers (rewriter.py:337-396).
    """
    by_source: dict[int, list[int]] = {}
    for n in g.nodes:
        if n.kind is NodeKind.SWAP_IN:
            by_source.setdefault(_only_read_input(g, n.id).src, []).append(n.id)

    def first_use(si: int) -> int:
        uses = [order[e.dst] for e in g.out_edges(si) if e.action is _READ]
        return min(uses) if uses else 0

    merged: dict[int, int] = {}
    for ids in by_source.values():
        if len(ids) < 2:
            continue
        keyed = sorted((first_use(si), si) for si in ids)
        clusters: list[list[tuple[int, int]]] = []
        for item in keyed:
            if clusters and item[0] - clusters[-1][0][0] <= distance_threshold:
                clusters[-1].append(item)
            else:
                clusters.append([item])
        for cl in clusters:
            if len(cl) > 1:
                keep = min(si for _, si in cl)
                for _, si in cl:
                    if si != keep:
                        merged[si] = keep
    return _merge_into(g, merged)


# -- control-stage cycle check ------------------------------------------------------

class _Reach:
    """``reachable(cur, si)`` membership for the cumulative control stage.

    ``cur`` = query graph + control edges attached so far.  Descendant
    bitsets of the query graph are computed once; a query closes them over
    the attached control edges (each edge c->s contributes desc(s) once c is
    reached).  Falls back to explicit search when the query graph's
    read/control relation is cyclic.
    """

    def __init__(self, g: CompGraph):
        self.g = g
        nbi = g.node_by_id
        self.bit = {nid: i for i, nid in enumerate(nbi)}
        succs: dict[int, list[int]] = {nid: [] for nid in nbi}
        indeg = dict.fromkeys(nbi, 0)
        for e in g.edges:
            if e.action is _UPDATE or e.src not in nbi or e.dst not in nbi:
                continue
            succs[e.src].append(e.dst)
            indeg[e.dst] += 1
        topo = []
        ready = [nid for nid, d in indeg.items() if d == 0]
        while ready:
            nid = ready.pop()
            topo.append(nid)
            for s in succs[nid]:
                indeg[s] -= 1
                if indeg[s] == 0:
                    ready.append(s)
        self.desc = None
        if len(topo) == len(nbi):
            desc: dict[int, int] = {}
            bit = self.bit
            for nid in reversed(topo):
                acc = 1 << bit[nid]
                for s in succs[nid]:
                    acc |= desc[s]
                desc[nid] = acc
            self.desc = desc
        self.extra: list[tuple[int, int]] = []

    def add(self, c: int, s: int):
        self.extra.append((c, s))

    def reaches(self, start: int, goal: int) -> bool:
        if self.desc is None:
            return self._search(start, goal)
        bit = self.bit
        r = self.desc[start]
        pending = list(self.extra)
        grew = True
        while grew and pending:
            grew = False
            rest = []
            for c, s in pending:
                if (r >> bit[c]) & 1:
                    r |= self.desc[s]
                    grew = True
                else:
                    rest.append((c, s))
            pending = rest
        return (r >> bit[goal]) & 1 == 1

    def _search(self, start: int, goal: int) -> bool:
        g = self.g
        extra: dict[int, list[int]] = {}
        for c, s in self.extra:
            extra.setdefault(c, []).append(s)
        seen = {start}
        stack = [start]
        while stack:
            cur = stack.pop()
            if cur == goal:
                return True
            nxt = [e.dst for e in g.out_edges(cur) if e.action is not _UPDATE
                   and e.dst in g.node_by_id] + extra.get(cur, [])
            for d in nxt:
                if d not in seen:
                    seen.add(d)
                    stack.append(d)
        return False


# -- the pipeline -----------------------------------------------------------------

def _staged(name: str, fn, *args):
    try:
        return fn(*args)
    except RewriteError:
        raise
    except Exception as exc:
        raise RewriteError(f"stage {name!r}: {exc}") from exc


def _insert_all(g: CompGraph, picked) -> CompGraph:
    """All swap pairs in one sweep; ids as if inserted one at a time."""
    if not picked:
        return g
    nxt_node = g.max_node_id() + 1
    nxt_tensor = g.max_tensor_id() + 1
    edges = list(g.edges)
    # multiset removal, as repeated list.remove() would do
    remove: dict[EdgeRec, int] = {}
    nodes = list(g.nodes)
    tensors = list(g.tensors)
    tbi = g.tensor_by_id
    for edge, _ in picked:
        remove[edge] = remove.get(edge, 0) + 1
        so, si, new_t = _swap_pair_records(tbi[edge.tensor], edge.dst, nxt_node, nxt_tensor)
        nodes += (so, si)
        tensors += new_t
        edges += (EdgeRec(edge.src, so.id, _READ, edge.tensor),
                  EdgeRec(so.id, si.id, _READ, new_t[0].id),
                  EdgeRec(si.id, edge.dst, _READ, new_t[1].id))
        nxt_node += 2
        nxt_tensor += 2
    kept = []
    for e in edges[:len(g.edges)]:
        left = remove.get(e)
        if left:
            remove[e] = left - 1
        else:
            kept.append(e)
    return CompGraph(nodes, kept + edges[len(g.edges):], tensors)


def rewrite(g: CompGraph, cfg: RewriteConfig) -> tuple[CompGraph, RewriteReport]:
    """Full pipeline: phases, order, select, insert, fuse, control, validate.

    Deterministic for a given (graph, config), inserted ids included.  Graphs
    that already contain swap nodes are refused (rewriter.py:407-489).
    """
    report = RewriteReport()
    if any(n.kind in SWAP_KINDS for n in g.nodes):
        raise RewriteError("stage 'precheck': graph already contains swap nodes; "
                           "rewrite must start from an unrewritten graph")
    if not _phases_resolvable(g, cfg):
        raise RewriteError("stage 'phases': no phase tags and no optimizer_scopes; "
                           "cannot tell forward from backward")

    tagged = _staged("phases", resolve_phases, g, cfg.optimizer_scopes)
    base_order = _staged("order", topo_order, tagged)
    picked = _staged("select", select_candidates, tagged, base_order, cfg, report)

    cur = _staged("insert", _insert_all, tagged, picked)
    report.edges_rewritten.extend((e.src, e.dst, tid) for e, tid in picked)
    cur = _staged("fuse_swap_outs", fuse_swap_outs, cur)
    if cfg.fuse_swapins:
        cur = _staged("fuse_swap_ins", fuse_swap_ins, cur, base_order, cfg.swapin_fuse_distance)

    if picked:
        # every query sees the post-fusion graph without earlier attachments
        q_graph = cur
        q_order = _staged("order", topo_order, q_graph)
        index = _staged("ctrl_select", ctrl.CtrlIndex, q_graph, q_order)
        pick = index.direct_order if cfg.ctrld_strategy == "direct_order" else index.chain_rule
        reach = _Reach(q_graph)
        added: list[EdgeRec] = []
        for si in [n.id for n in q_graph.nodes if n.kind is NodeKind.SWAP_IN]:
            so_edge = _only_read_input(q_graph, si)
            users = [e.dst for e in q_graph.out_edges(si) if e.action is _READ]
            if not users:
                report.skipped.append({"reason": "swap-in has no consumer", "node": si})
                continue
            target = min(users, key=lambda nid: (q_order[nid], nid))
            q = ctrl.CtrlQuery(source=so_edge.src, target=target, lb=cfg.lb, ub=cfg.ub)
            chosen = _staged("ctrl_select", pick, q)
            if chosen is None:
                chosen = _staged("ctrl_select", index.fallback, so_edge.src, target)
                if chosen is not None:
                    report.skipped.append({"reason": "strategy found no control op; used fallback",
                                           "node": si, "control": chosen})
            if chosen is None:
                report.skipped.append({"reason": "no control op in window; swap-in left eager",
                                       "node": si})
                continue
            if reach.reaches(si, chosen):
                raise RewriteError(
                    f"stage 'attach_control': control edge {chosen} -> {si} would close a "
                    f"cycle ({chosen} is reachable from {si})")
            reach.add(chosen, si)
            added.append(EdgeRec(chosen, si, _CONTROL))
            report.control_edges_added += 1
        if added:
            cur = CompGraph(cur.nodes, cur.edges + tuple(added), cur.tensors)

    problems = _staged("validate", validate, cur)
    if problems:
        raise RewriteError(f"stage 'validate': rewritten graph is invalid: {problems[:3]}")

    report.tensors_swapped = len({tid for _, tid in picked})
    report.swap_outs_added = sum(1 for n in cur.nodes if n.kind is NodeKind.SWAP_OUT)
    report.swap_ins_added = sum(1 for n in cur.nodes if n.kind is NodeKind.SWAP_IN)
    log.info("rewrite: %d tensors swapped, %d swap-outs, %d swap-ins, %d control edges",
             report.tensors_swapped, report.swap_outs_added, report.swap_ins_added,
             report.control_edges_added)
    return cur, report
