"""Control-operation strategies that decide when each swap-in fires.

Same contract as the reference (``swapgraph/control.py``): a ``CtrlQuery``
names the swap-out (window floor) and the consumer the swap-in feeds; a
strategy returns the id of an op from which the consumer is reachable, or
None.  The rewriter then adds ``op -control-> swap_in`` and, at run time, the
executor issues the host->device copy when that op's completion event fires.

Implementation differs from the reference: :class:`CtrlIndex` precomputes,
once per (graph, order), the ancestor relation as integer bitsets, the
per-level lists of eligible ops and memoised swap-transparent successor
lists, so each query is O(window) instead of O(V+E)
(reference: ``ancestors`` per query, ``control.py:82``, ``:119``).

Reference anchors: ``CtrlQuery`` control.py:26-39, ``_logical_successors``
:42-62, ``_eligible`` :65-69, ``direct_order`` (paper Alg. 1) :72-93,
``_bfs_seed`` :96-108, ``chain_rule`` (paper Alg. 2) :111-147,
``fallback_control`` :150-155, ``attach_control`` :158-169.
"""

from __future__ import annotations

from dataclasses import dataclass

from .graph import (
    CompGraph,
    EdgeAction,
    EdgeRec,
    Phase,
    SWAP_KINDS,
    ancestors,
    reachable,
)


@dataclass(frozen=True)
class CtrlQuery:
    """Search window for one swap-in.

    ``source`` is the window floor (the swap-out, or the producer for an
    unrewritten graph); ``target`` is the consumer fed by the swap-in;
    ``lb``/``ub`` bound the distance between the chosen op and the target.
    """

    source: int
    target: int
    lb: int = 1
    ub: int = 10000


class CtrlIndex:
    """Query accelerator for one (graph, order) pair.

    Answers are identical to the reference's per-query formulation; only the
    cost changes.  ``ancestor_of(a, b)`` is "b reachable from a over
    read/control edges".  When the read/control relation is not a DAG
    (possible only through edges into parameterized nodes, which
    ``topo_order`` ignores) the index falls back to explicit closures.
    """

    def __init__(self, g: CompGraph, order: dict[int, int]):
        self.g = g
        self.order = order
        nbi = g.node_by_id
        self._succ_memo: dict[int, list[int]] = {}
        self._anc_sets: dict[int, set[int]] = {}
        # eligible control ops per order level, ascending id (control.py:65-69)
        levels: dict[int, list[int]] = {}
        for n in g.nodes:  # ascending id
            if not n.parameterized and n.kind not in SWAP_KINDS:
                levels.setdefault(order[n.id], []).append(n.id)
        self._levels = levels
        self._bit = {nid: i for i, nid in enumerate(nbi)}
        self._anc = self._ancestor_bits()

    def _ancestor_bits(self):
        """anc[v] = bitset of nodes that reach v; None if not a DAG."""
        g = self.g
        nbi = g.node_by_id
        bit = self._bit
        preds: dict[int, list[int]] = {nid: [] for nid in nbi}
        indeg = dict.fromkeys(nbi, 0)
        succs: dict[int, list[int]] = {nid: [] for nid in nbi}
        for e in g.edges:
            if e.action is EdgeAction.UPDATE or e.src not in nbi or e.dst not in nbi:
                continue
            preds[e.dst].append(e.src)
            succs[e.src].append(e.dst)
            indeg[e.dst] += 1
        anc: dict[int, int] = {}
        ready = [nid for nid, d in indeg.items() if d == 0]
        while ready:
            nid = ready.pop()
            acc = 1 << bit[nid]
            for p in preds[nid]:
                acc |= anc[p]
            anc[nid] = acc
            for s in succs[nid]:
                indeg[s] -= 1
                if indeg[s] == 0:
                    ready.append(s)
        if len(anc) != len(nbi):
            return None
        return anc

    def reaches(self, src: int, target: int) -> bool:
        """True if ``target`` is reachable from ``src`` (or src == target)."""
        if self._anc is not None:
            return (self._anc[target] >> self._bit[src]) & 1 == 1
        s = self._anc_sets.get(target)
        if s is None:
            s = self._anc_sets[target] = ancestors(self.g, target)
        return src in s

    def logical_successors(self, nid: int) -> list[int]:
        """Non-update successors with swap nodes looked through (control.py:42-62)."""
        got = self._succ_memo.get(nid)
        if got is not None:
            return got
        g = self.g
        nbi = g.node_by_id
        seen = {nid}
        found = []
        stack = [nid]
        while stack:
            for e in g.out_edges(stack.pop()):
                d = e.dst
                if e.action is EdgeAction.UPDATE or d in seen:
                    continue
                seen.add(d)
                if nbi[d].kind in SWAP_KINDS:
                    stack.append(d)
                else:
                    found.append(d)
        found.sort()
        self._succ_memo[nid] = found
        return found

    def bfs_seed(self, source: int) -> int:
        """Walk back from a swap node to the op whose value it forwards (control.py:96-108)."""
        g = self.g
        cur = source
        for _ in range(len(g.nodes) + 1):
            if g.node_by_id[cur].kind not in SWAP_KINDS:
                return cur
            reads = [e for e in g.in_edges(cur) if e.action is EdgeAction.READ]
            if len(reads) != 1:
                return cur
            cur = reads[0].src
        return cur

    def direct_order(self, q: CtrlQuery) -> int | None:
        """Paper Alg. 1: nearest-to-lb populated level, lowest id wins."""
        order = self.order
        t_level = order[q.target]
        floor = max(t_level - q.ub + 1, order[q.source])
        if q.target not in self.g.node_by_id:
            raise KeyError(f"unknown node id {q.target}")
        levels = self._levels
        for dist in range(q.lb, q.ub + 1):
            lv = t_level - dist
            if lv <= floor:
                return None
            for nid in levels.get(lv, ()):
                if self.reaches(nid, q.target):
                    return nid  # lists are ascending, first hit is the min
        return None

    def chain_rule(self, q: CtrlQuery) -> int | None:
        """Paper Alg. 2: level-synchronous walk of the forward phase."""
        g = self.g
        nbi = g.node_by_id
        order = self.order
        if q.target not in nbi:
            raise KeyError(f"unknown node id {q.target}")
        lo, hi = q.lb, q.ub
        frontier = [self.bfs_seed(q.source)]
        visited = set(frontier)
        fwd, bwd = Phase.FORWARD, Phase.BACKWARD
        while frontier:
            if hi == 0 or lo > hi:
                return None
            if lo <= 0:
                lo_o = order[q.source]
                hi_o = order[q.target]
                best = None
                for nid in frontier:
                    for s in self.logical_successors(nid):
                        if (nbi[s].phase is bwd and lo_o < order[s] < hi_o
                                and (best is None or s < best)
                                and self.reaches(s, q.target)):
                            best = s
                if best is not None:
                    return best
            nxt = []
            for nid in frontier:
                for s in self.logical_successors(nid):
                    if nbi[s].phase is fwd and s not in visited:
                        visited.add(s)
                        nxt.append(s)
            lo -= 1
            hi -= 1
            frontier = nxt
        return None

    def fallback(self, source: int, target: int) -> int | None:
        """Latest op below the target that reaches it (control.py:150-155)."""
        span = self.order[target] - self.order[source]
        if span <= 0:
            return None
        return self.direct_order(CtrlQuery(source=source, target=target, lb=1, ub=span))


def direct_order(g: CompGraph, order: dict[int, int], q: CtrlQuery) -> int | None:
    """Pick the control op by order distance alone (paper Alg. 1, control.py:72-93)."""
    return CtrlIndex(g, order).direct_order(q)


def chain_rule(g: CompGraph, order: dict[int, int], q: CtrlQuery) -> int | None:
    """Pick the control op by walking the forward phase (paper Alg. 2, control.py:111-147)."""
    return CtrlIndex(g, order).chain_rule(q)


def fallback_control(g: CompGraph, order: dict[int, int], source: int, target: int) -> int | None:
    """direct_order with lb=1, ub=span (control.py:150-155)."""
    return CtrlIndex(g, order).fallback(source, target)


def attach_control(g: CompGraph, ctrl: int, swap_in: int) -> CompGraph:
    """Return ``g`` plus ``ctrl -control-> swap_in``; refuses edges closing a cycle."""
    nbi = g.node_by_id
    if ctrl not in nbi or swap_in not in nbi:
        raise KeyError(f"unknown node in control edge {ctrl} -> {swap_in}")
    if nbi[swap_in].parameterized:
        raise ValueError(f"control edge into parameterized node {swap_in}")
    if ctrl in reachable(g, swap_in):
        raise ValueError(
            f"control edge {ctrl} -> {swap_in} would close a cycle "
            f"({ctrl} is reachable from {swap_in})")
    return CompGraph(g.nodes, g.edges + (EdgeRec(ctrl, swap_in, EdgeAction.CONTROL),), g.tensors)
