"""Serial float64 interpreter — restatement of ``swapgraph/interp.py``.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Semantics followed:

* ops run one at a time in ascending (order, id) among ready ops
  (interp.py:115-158); only ops reachable from parameterized nodes run
  (interp.py:84-95);
* operands are sorted by origin tensor id, the origin following
  swap/identity/assign_update chains (interp.py:29-50, :124);
* parameterized producers are read live from the variable state
  (interp.py:129-131); update edges commit right after their producer runs
  (interp.py:140-151);
* swap nodes are identities that hand the same array on (interp.py:168-170);
* vocabulary add/sub/mul/neg/matmul/identity/assign_update with the
  reference's shape errors (interp.py:166-195).

Works on any graph object with the reference's interface (ours or theirs).
"""

from __future__ import annotations

import heapq

import numpy as np

_PASS = ("identity", "assign_update")


def _topo(g):
    # local ASAP levels (graph.py:341-378) so the oracle does not depend on
    # the product's ordering code
    level = {}
    preds = {n.id: [] for n in g.nodes}
    for e in g.edges:
        d = g.node_by_id.get(e.dst)
        if d is None or e.src not in g.node_by_id or d.parameterized:
            continue
        preds[e.dst].append(e.src)
    remaining = set(preds)
    while remaining:
        progressed = False
        for nid in sorted(remaining):
            if all(p in level for p in preds[nid]):
                node = g.node_by_id[nid]
                level[nid] = 0 if node.parameterized else 1 + max((level[p] for p in preds[nid]), default=0)
                remaining.discard(nid)
                progressed = True
        if not progressed:
            raise ValueError("cyclic graph")
    return level


def _kind(n):
    return n.kind.value if hasattr(n.kind, "value") else str(n.kind)


def _action(e):
    return e.action.value if hasattr(e.action, "value") else str(e.action)


def origin_of(g, tid, memo):
    """Originally produced tensor behind swap/identity chains (interp.py:29-50)."""
    path = []
    cur = tid
    while cur not in memo:
        path.append(cur)
        prod = g.node_by_id[g.tensor_by_id[cur].producer]
        passes = _kind(prod) in ("swap_out", "swap_in") or (_kind(prod) == "compute" and prod.name in _PASS)
        if not passes:
            break
        reads = [e for e in g.in_edges(prod.id) if _action(e) == "read"]
        if len(reads) != 1 or reads[0].tensor in path:
            break
        cur = reads[0].tensor
    root = memo.get(cur, cur)
    for t in path:
        memo[t] = root
    return root


def apply_op(node, args):
    kind = _kind(node)
    name = node.name

    def arity(n):
        if len(args) != n:
            raise ValueError(f"{name!r} (node {node.id}) expects {n} input(s), got {len(args)}")

    if kind in ("swap_out", "swap_in") or name in _PASS:
        arity(1)
        return args[0]
    if name == "neg":
        arity(1)
        return -args[0]
    if name in ("add", "sub", "mul"):
        arity(2)
        a, b = args
        if a.shape != b.shape:
            raise ValueError(f"{name} (node {node.id}): shapes {a.shape} and {b.shape} differ")
        return a + b if name == "add" else (a - b if name == "sub" else a * b)
    if name == "matmul":
        arity(2)
        a, b = args
        if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
            raise ValueError(f"matmul (node {node.id}): shapes {a.shape} @ {b.shape} invalid")
        return a @ b
    raise ValueError(f"unsupported op {name!r} (node {node.id})")


def schedule(g):
    """(runnable set, serial op sequence) exactly as the interpreter would run them."""
    order = _topo(g)
    runnable = set()
    seen = {n.id for n in g.nodes if n.parameterized}
    stack = list(seen)
    while stack:
        nid = stack.pop()
        for e in g.out_edges(nid):
            if _action(e) == "update" or e.dst in seen:
                continue
            seen.add(e.dst)
            stack.append(e.dst)
            if not g.node_by_id[e.dst].parameterized:
                runnable.add(e.dst)
    pending = {}
    for nid in runnable:
        c = 0
        for e in g.in_edges(nid):
            if _action(e) == "read":
                if not g.node_by_id[g.tensor_by_id[e.tensor].producer].parameterized:
                    c += 1
            elif _action(e) == "control" and e.src in runnable:
                c += 1
        pending[nid] = c
    heap = [(order[n], n) for n in runnable if pending[n] == 0]
    heapq.heapify(heap)
    seq = []
    while heap:
        _, nid = heapq.heappop(heap)
        seq.append(nid)
        wake = [e.dst for e in g.out_edges(nid) if _action(e) == "control" and e.dst in runnable]
        for t in g.produced_tensors(nid):
            wake += [e.dst for e in g.consumer_edges(t.id) if _action(e) == "read" and e.dst in runnable]
        for d in wake:
            pending[d] -= 1
            if pending[d] == 0:
                heapq.heappush(heap, (order[d], d))
    return runnable, seq


def interpret(g, inputs):
    """Final state of every parameterized node, float64 (interp.py:58-163)."""
    state = {}
    for n in g.nodes:
        if not n.parameterized:
            continue
        if n.name in inputs:
            state[n.id] = np.asarray(inputs[n.name], dtype=np.float64)
        elif _kind(n) == "constant":
            try:
                state[n.id] = np.asarray(float(n.name), dtype=np.float64)
            except ValueError:
                raise ValueError(f"constant {n.name!r} (node {n.id}) is unbound "
                                 f"and its name is not a number") from None
        else:
            raise ValueError(f"variable {n.name!r} (node {n.id}) is unbound")
    runnable, seq = schedule(g)
    memo = {}
    values = {}
    for nid in seq:
        node = g.node_by_id[nid]
        reads = sorted((e for e in g.in_edges(nid) if _action(e) == "read"),
                       key=lambda e: (origin_of(g, e.tensor, memo), e.tensor))
        args = []
        for e in reads:
            prod = g.tensor_by_id[e.tensor].producer
            args.append(state[prod] if g.node_by_id[prod].parameterized else values[e.tensor])
        out = apply_op(node, args)
        produced = g.produced_tensors(nid)
        if len(produced) > 1:
            raise ValueError(f"op {node.name!r} (node {nid}) has multiple outputs; "
                             "the interpreter vocabulary is single-output")
        for t in produced:
            values[t.id] = out
        for e in g.out_edges(nid):
            if _action(e) != "update":
                continue
            var = g.node_by_id[e.dst]
            if not var.parameterized:
                raise ValueError(f"update edge into non-variable node {e.dst}")
            if state[e.dst].shape != values[e.tensor].shape:
                raise ValueError(f"update into {var.name!r}: shape {values[e.tensor].shape} "
                                 f"!= {state[e.dst].shape}")
            state[e.dst] = values[e.tensor]
    if len(seq) != len(runnable):
        raise ValueError(f"ops never became ready (missing inputs?): {sorted(runnable - set(seq))}")
    return {g.node_by_id[nid].name: v for nid, v in state.items()}
