"""Graph IR for the swap rewriter: ops, tensors and labelled edges.

Drop-in for the reference IR (``swapgraph/graph.py``): the record types,
enum values, canonical ordering, ``topo_order`` levels, reachability,
``lifetime`` and the ``validate`` violation codes are the same, so a graph
built with the reference constructors and one built here serialise to the
same bytes.  What differs is the implementation:

* ``CompGraph`` builds its adjacency indices lazily, on first query, so the
  rewriter can construct a graph once at the end instead of after every edit
  (the reference rebuilds on every insert/attach, ``graph.py:119-140``).
* ``topo_order`` is a level-by-level Kahn sweep over dense integer arrays.

Reference anchors: records ``graph.py:38-92``, canonical edge key
``graph.py:95-96``, ``CompGraph`` ``graph.py:99-186``, ``validate``
``graph.py:254-338``, ``topo_order`` ``graph.py:341-378``,
``reachable``/``ancestors`` ``graph.py:393-424``, ``lifetime``
``graph.py:427-446``.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass
from enum import Enum

log = logging.getLogger("swapgraph")

HOST = "host"
_ACC_PREFIX = "acc:"


def accelerator(index: int = 0) -> str:
    """Device label of accelerator ``index`` (``acc:<index>``)."""
    return _ACC_PREFIX + str(index)


def is_accelerator(device: str) -> bool:
    return device.startswith(_ACC_PREFIX)


def is_valid_device(device: str) -> bool:
    """``host`` or ``acc:<decimal digits>`` (graph.py:29-35)."""
    if device == HOST:
        return True
    return is_accelerator(device) and device[len(_ACC_PREFIX):].isdigit()


class NodeKind(str, Enum):
    COMPUTE = "compute"
    VARIABLE = "variable"
    CONSTANT = "constant"
    SWAP_OUT = "swap_out"
    SWAP_IN = "swap_in"


class Phase(str, Enum):
    FORWARD = "forward"
    BACKWARD = "backward"
    UPDATE = "update"
    UNKNOWN = "unknown"


class EdgeAction(str, Enum):
    READ = "read"
    UPDATE = "update"
    CONTROL = "control"


PARAM_KINDS = frozenset((NodeKind.VARIABLE, NodeKind.CONSTANT))
SWAP_KINDS = frozenset((NodeKind.SWAP_OUT, NodeKind.SWAP_IN))


@dataclass(frozen=True)
class OpNode:
    """One operation; ``parameterized`` is true exactly for variables/constants."""

    id: int
    name: str
    scope: str = ""
    kind: NodeKind = NodeKind.COMPUTE
    parameterized: bool = False
    phase: Phase = Phase.UNKNOWN
    device: str = "acc:0"
    cost_hint: float = 1.0


@dataclass(frozen=True)
class TensorSpec:
    id: int
    producer: int
    size_bytes: int = 0
    dtype: str = "f32"


@dataclass(frozen=True)
class EdgeRec:
    """Labelled edge; ``tensor`` is set for read/update edges, None for control."""

    src: int
    dst: int
    action: EdgeAction = EdgeAction.READ
    tensor: int | None = None


def edge_sort_key(e: EdgeRec) -> tuple:
    """Canonical edge order: (src, dst, action value, tensor or -1)."""
    t = e.tensor
    return (e.src, e.dst, e.action.value, -1 if t is None else t)


def _node_key(n: OpNode) -> int:
    return n.id


def _tensor_key(t: TensorSpec) -> int:
    return t.id


class CompGraph:
    """Immutable graph value.

    Collections are normalised (sorted) on construction so equal content
    compares equal whatever the build order.  Adjacency indices are derived
    on first use and cached on the instance.
    """

    __slots__ = ("nodes", "edges", "tensors", "node_by_id", "tensor_by_id",
                 "_out", "_in", "_produced", "_consumers")

    def __init__(self, nodes, edges, tensors):
        self.nodes: tuple[OpNode, ...] = tuple(sorted(nodes, key=_node_key))
        self.edges: tuple[EdgeRec, ...] = tuple(sorted(edges, key=edge_sort_key))
        self.tensors: tuple[TensorSpec, ...] = tuple(sorted(tensors, key=_tensor_key))
        self.node_by_id = {n.id: n for n in self.nodes}
        self.tensor_by_id = {t.id: t for t in self.tensors}
        self._out = None
        self._in = None
        self._produced = None
        self._consumers = None

    # -- lazily derived indices -------------------------------------------
    def _index_edges(self):
        out = {nid: [] for nid in self.node_by_id}
        inc = {nid: [] for nid in self.node_by_id}
        cons = {tid: [] for tid in self.tensor_by_id}
        for e in self.edges:
            # dangling endpoints are kept; validate() reports them
            lst = out.get(e.src)
            if lst is None:
                lst = out[e.src] = []
            lst.append(e)
            lst = inc.get(e.dst)
            if lst is None:
                lst = inc[e.dst] = []
            lst.append(e)
            if e.tensor is not None:
                lst = cons.get(e.tensor)
                if lst is None:
                    lst = cons[e.tensor] = []
                lst.append(e)
        self._out, self._in, self._consumers = out, inc, cons

    def _index_tensors(self):
        prod = {nid: [] for nid in self.node_by_id}
        for t in self.tensors:
            prod.setdefault(t.producer, []).append(t)
        self._produced = prod

    # -- queries (same surface as the reference) -----------------------------
    def node(self, node_id: int) -> OpNode:
        return self.node_by_id[node_id]

    def tensor(self, tensor_id: int) -> TensorSpec:
        return self.tensor_by_id[tensor_id]

    def out_edges(self, node_id: int) -> list[EdgeRec]:
        if self._out is None:
            self._index_edges()
        return self._out.get(node_id, [])

    def in_edges(self, node_id: int) -> list[EdgeRec]:
        if self._in is None:
            self._index_edges()
        return self._in.get(node_id, [])

    def produced_tensors(self, node_id: int) -> list[TensorSpec]:
        if self._produced is None:
            self._index_tensors()
        return self._produced.get(node_id, [])

    def consumer_edges(self, tensor_id: int) -> list[EdgeRec]:
        """Read/update edges carrying ``tensor_id``."""
        if self._consumers is None:
            self._index_edges()
        return self._consumers.get(tensor_id, [])

    def is_parameterized(self, node_id: int) -> bool:
        return self.node_by_id[node_id].parameterized

    def max_node_id(self) -> int:
        return self.nodes[-1].id if self.nodes else -1

    def max_tensor_id(self) -> int:
        return self.tensors[-1].id if self.tensors else -1

    def __eq__(self, other) -> bool:
        if not isinstance(other, CompGraph):
            return NotImplemented
        return (self.nodes == other.nodes and self.edges == other.edges
                and self.tensors == other.tensors)

    def __hash__(self):
        return hash((self.nodes, self.edges, self.tensors))

    def __repr__(self) -> str:
        return (f"CompGraph(nodes={len(self.nodes)}, edges={len(self.edges)}, "
                f"tensors={len(self.tensors)})")


# -- convenience constructors (graph.py:189-204) ---------------------------

def variable_node(node_id: int, name: str, *, scope: str = "", device: str = "acc:0") -> OpNode:
    return OpNode(node_id, name, scope, NodeKind.VARIABLE, True, Phase.UNKNOWN, device, 0.0)


def constant_node(node_id: int, name: str, *, scope: str = "", device: str = "acc:0") -> OpNode:
    return OpNode(node_id, name, scope, NodeKind.CONSTANT, True, Phase.UNKNOWN, device, 0.0)


def compute_node(node_id: int, name: str, *, scope: str = "", phase: Phase = Phase.UNKNOWN,
                 device: str = "acc:0", cost_hint: float = 1.0) -> OpNode:
    return OpNode(node_id, name, scope, NodeKind.COMPUTE, False, phase, device, cost_hint)


class CycleError(ValueError):
    """The execution subgraph has a cycle; ``cycle`` lists it (first id repeated)."""

    def __init__(self, cycle: list[int]):
        self.cycle = cycle
        super().__init__("execution subgraph contains a cycle: " + " -> ".join(map(str, cycle)))


@dataclass(frozen=True)
class Violation:
    code: str
    message: str
    node: int | None = None
    edge: EdgeRec | None = None
    tensor: int | None = None


# -- ordering ---------------------------------------------------------------

def execution_adjacency(g: CompGraph):
    """Predecessor/successor lists of the execution subgraph.

    Update edges into variables are dropped, and no incoming edge moves a
    parameterized node (graph.py:224-230, :355-357).
    """
    nbi = g.node_by_id
    preds = {nid: [] for nid in nbi}
    succs = {nid: [] for nid in nbi}
    for e in g.edges:
        d = nbi.get(e.dst)
        # an edge into a parameterized node (update edges included) never
        # moves it off level 0; update edges into compute ops do count
        if d is None or e.src not in nbi or d.parameterized:
            continue
        preds[e.dst].append(e.src)
        succs[e.src].append(e.dst)
    return preds, succs


def topo_order(g: CompGraph) -> dict[int, int]:
    """ASAP level of every node (graph.py:341-378).

    Parameterized nodes sit at 0; any other node is one past its latest
    read/control predecessor.  Raises :class:`CycleError` if no order exists.
    """
    preds, succs = execution_adjacency(g)
    indeg = {nid: len(p) for nid, p in preds.items()}
    order: dict[int, int] = {}
    frontier = [nid for nid, d in indeg.items() if d == 0]
    nbi = g.node_by_id
    while frontier:
        nxt = []
        for nid in frontier:
            if nbi[nid].parameterized:
                order[nid] = 0
            else:
                best = 0
                for p in preds[nid]:
                    v = order[p]
                    if v > best:
                        best = v
                order[nid] = best + 1
            for s in succs[nid]:
                indeg[s] -= 1
                if indeg[s] == 0:
                    nxt.append(s)
        frontier = nxt
    if len(order) != len(indeg):
        left = {nid for nid in indeg if nid not in order}
        raise CycleError(_cycle_in(succs, left))
    return order


def _cycle_in(succs, left: set[int]) -> list[int]:
    """Walk from the smallest blocked id along smallest blocked successors."""
    pos: dict[int, int] = {}
    walk: list[int] = []
    cur = min(left)
    while cur not in pos:
        pos[cur] = len(walk)
        walk.append(cur)
        # StopIteration escapes when a blocked node has no blocked successor,
        # exactly as the reference's next() does (graph.py:437-446)
        cur = next(s for s in sorted(succs[cur]) if s in left)
    return walk[pos[cur]:] + [cur]


# -- reachability -----------------------------------------------------------

def reachable(g: CompGraph, src: int) -> set[int]:
    """Nodes reachable from ``src`` over read/control edges (``src`` included)."""
    if src not in g.node_by_id:
        raise KeyError(f"unknown node id {src}")
    return _closure(g, src, forward=True)


def ancestors(g: CompGraph, dst: int) -> set[int]:
    """Nodes that reach ``dst`` over read/control edges (``dst`` included)."""
    if dst not in g.node_by_id:
        raise KeyError(f"unknown node id {dst}")
    return _closure(g, dst, forward=False)


def _closure(g: CompGraph, start: int, forward: bool) -> set[int]:
    nbi = g.node_by_id
    upd = EdgeAction.UPDATE
    adj = g.out_edges if forward else g.in_edges
    seen = {start}
    stack = [start]
    while stack:
        for e in adj(stack.pop()):
            if e.action is upd:
                continue
            nxt = e.dst if forward else e.src
            if nxt not in seen and nxt in nbi:
                seen.add(nxt)
                stack.append(nxt)
    return seen


def lifetime(g: CompGraph, order: dict[int, int], tensor_id: int) -> int:
    """Order steps a tensor stays live past its producer (PAPER §3.5).

    Read consumers hold it until their own step; update edges commit at the
    producer's step.  Unconsumed tensors have lifetime 0 (graph.py:427-446).
    """
    t = g.tensor_by_id[tensor_id]
    uses = g.consumer_edges(tensor_id)
    if not uses:
        log.warning("tensor %d has no consumers; lifetime defaults to 0", tensor_id)
        return 0
    born = order[t.producer]
    last = born
    for e in uses:
        if e.action is EdgeAction.READ and order[e.dst] > last:
            last = order[e.dst]
    return last - born


# -- validation ---------------------------------------------------------------

def _passes_value(n: OpNode) -> bool:
    return n.kind in SWAP_KINDS or (n.kind is NodeKind.COMPUTE and n.name == "identity")


def _source_forwards(g: CompGraph, src: int, producer: int) -> bool:
    """``src`` is the producer or forwards its value through swap/identity ops."""
    cur = src
    for _ in range(len(g.nodes) + 1):
        if cur == producer:
            return True
        n = g.node_by_id.get(cur)
        if n is None or not _passes_value(n):
            return False
        reads = [e for e in g.in_edges(cur) if e.action is EdgeAction.READ]
        if len(reads) != 1:
            return False
        cur = reads[0].src
    return False


def validate(g: CompGraph) -> list[Violation]:
    """All structural violations (graph.py:254-338); empty means valid."""
    found: list[Violation] = []
    add = found.append
    nbi, tbi = g.node_by_id, g.tensor_by_id

    ids: set[int] = set()
    for n in g.nodes:
        if n.id in ids:
            add(Violation("dup-node-id", f"node id {n.id} appears more than once", node=n.id))
        ids.add(n.id)
        if not is_valid_device(n.device):
            add(Violation("bad-device", f"node {n.id} has malformed device {n.device!r}", node=n.id))
        if n.kind in SWAP_KINDS and n.device != HOST:
            add(Violation("swap-off-host", f"swap node {n.id} must be placed on host", node=n.id))
        if (n.kind in PARAM_KINDS) != n.parameterized:
            add(Violation("param-kind-mismatch",
                          f"node {n.id} kind {n.kind.value} disagrees with "
                          f"parameterized={n.parameterized}", node=n.id))
        if n.cost_hint < 0:
            add(Violation("bad-cost", f"node {n.id} has negative cost_hint", node=n.id))

    tids: set[int] = set()
    for t in g.tensors:
        if t.id in tids:
            add(Violation("dup-tensor-id", f"tensor id {t.id} appears more than once", tensor=t.id))
        tids.add(t.id)
        if t.producer not in nbi:
            add(Violation("no-producer", f"tensor {t.id} names unknown producer {t.producer}",
                          tensor=t.id))
        if t.size_bytes < 0:
            add(Violation("bad-size", f"tensor {t.id} has negative size_bytes", tensor=t.id))

    for e in g.edges:
        if e.src not in nbi or e.dst not in nbi:
            add(Violation("dangling-edge", f"edge {e} references an unknown node", edge=e))
            continue
        if e.src == e.dst:
            add(Violation("self-loop", f"node {e.src} has a self-loop", edge=e))
        dst = nbi[e.dst]
        if e.action is EdgeAction.CONTROL:
            if e.tensor is not None:
                add(Violation("control-with-tensor", f"control edge {e} must not carry a tensor",
                              edge=e))
            if dst.parameterized:
                add(Violation("control-to-variable", f"control edge into parameterized node {dst.id}",
                              edge=e))
            continue
        if e.tensor is None:
            add(Violation("data-without-tensor", f"{e.action.value} edge {e} carries no tensor",
                          edge=e))
            continue
        t = tbi.get(e.tensor)
        if t is None:
            add(Violation("unknown-tensor", f"edge {e} references unknown tensor {e.tensor}", edge=e))
            continue
        if t.producer in nbi and not _source_forwards(g, e.src, t.producer):
            add(Violation("wrong-source",
                          f"edge {e} carries tensor {t.id} but src {e.src} is not its producer "
                          f"or a swap/identity chain from it", edge=e))
        if e.action is EdgeAction.UPDATE and dst.kind is not NodeKind.VARIABLE:
            add(Violation("update-to-nonvariable", f"update edge {e} into non-variable node {dst.id}",
                          edge=e))

    try:
        topo_order(g)
    except CycleError as exc:
        add(Violation("cycle", str(exc)))

    # reachable non-parameterized nodes need a read input or they never fire
    live = {n.id for n in g.nodes if n.parameterized}
    stack = list(live)
    while stack:
        for e in g.out_edges(stack.pop()):
            if e.action is not EdgeAction.UPDATE and e.dst not in live and e.dst in nbi:
                live.add(e.dst)
                stack.append(e.dst)
    for nid in sorted(live):
        if nbi[nid].parameterized:
            continue
        if not any(e.action is EdgeAction.READ for e in g.in_edges(nid)):
            add(Violation("no-data-input", f"reachable node {nid} has no incoming read edge",
                          node=nid))
    return found
