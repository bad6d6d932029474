"""Interpreter-vocabulary training graphs (BASELINE config 1).

``ffchain(L, N)`` is a feed-forward chain of ``L`` N×N ``matmul`` layers
with a backward pass in the same vocabulary and one ``sub`` update per
weight — the graph the reference CPU executor (``interp.py:58-190``) and the
GPU executor both run.  Shape of one step:

    forward   h[i+1] = matmul(h[i], W[i])            i = 0..L-1, h[0] = x
    backward  g[L]   = neg(h[L])
              dW[i]  = mul(g[i+1], h[i+1])           elementwise
              g[i]   = matmul(g[i+1], W[i])          i = L-1..1
    update    W[i]  <- sub(W[i], dW[i])              update edge into W[i]

Every activation h[1..L] is read forward->backward, so a default rewrite
swaps all ``L`` of them.  Inputs: ``numpy.random.default_rng(seed)``
standard normal × ``scale`` per variable.
"""

from __future__ import annotations

import numpy as np

from .graph import CompGraph, EdgeAction, EdgeRec, NodeKind, OpNode, Phase, TensorSpec


def ffchain(layers: int, n: int, elem_bytes: int = 4) -> CompGraph:
    if layers < 1 or n < 1:
        raise ValueError("ffchain needs layers >= 1 and n >= 1")
    nbytes = n * n * elem_bytes
    dtype = {4: "f32", 8: "f64"}.get(elem_bytes, f"b{elem_bytes}")
    nodes: list[OpNode] = []
    edges: list[EdgeRec] = []
    tensors: list[TensorSpec] = []

    def node(name, scope, kind=NodeKind.COMPUTE, phase=Phase.UNKNOWN, size=nbytes):
        nid = len(nodes)
        param = kind in (NodeKind.VARIABLE, NodeKind.CONSTANT)
        nodes.append(OpNode(nid, name, scope, kind, param, phase, "acc:0",
                            0.0 if param else 1.0))
        tensors.append(TensorSpec(len(tensors), nid, size, dtype))
        return nid, len(tensors) - 1

    def read(tid, dst):
        edges.append(EdgeRec(tensors[tid].producer, dst, EdgeAction.READ, tid))

    _, h = node("x", "input", NodeKind.VARIABLE)
    weights = []
    for i in range(layers):
        weights.append(node(f"W{i}", f"params/l{i}", NodeKind.VARIABLE))
    acts = [h]
    for i in range(layers):
        nid, h = node("matmul", f"model/l{i}", phase=Phase.FORWARD)
        read(acts[-1], nid)
        read(weights[i][1], nid)
        acts.append(h)
    nid, g = node("neg", "grads/top", phase=Phase.BACKWARD)
    read(acts[layers], nid)
    for i in reversed(range(layers)):
        nid, dw = node("mul", f"grads/l{i}/dw", phase=Phase.BACKWARD)
        read(g, nid)
        read(acts[i + 1], nid)
        unid, upd = node("sub", f"optimizer/l{i}", phase=Phase.UPDATE)
        read(weights[i][1], unid)
        read(dw, unid)
        edges.append(EdgeRec(unid, weights[i][0], EdgeAction.UPDATE, upd))
        if i > 0:
            nid, g2 = node("matmul", f"grads/l{i}/dx", phase=Phase.BACKWARD)
            read(g, nid)
            read(weights[i][1], nid)
            g = g2
    return CompGraph(nodes, edges, tensors)


def ffchain_inputs(g: CompGraph, n: int, seed: int = 0, scale: float = 0.1) -> dict[str, np.ndarray]:
    """float64 N×N per variable, drawn in ascending node id order."""
    rng = np.random.default_rng(seed)
    return {nd.name: rng.standard_normal((n, n)) * scale for nd in g.nodes if nd.parameterized}
