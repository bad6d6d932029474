"""Interpreter-vocabulary training graphs (BASELINE config 1).

``ffchain(L, N)`` is a feed-forward chain of ``L`` N×N ``matmul`` layers
with its backward pass written in the same vocabulary and one ``sub`` update
per weight — the graph the reference CPU executor (``interp.py:58-190``) and
the GPU executor both run.  The backward mirrors real autodiff: each
activation is re-read by two backward ops, and the op that consumes layer
i+1's activation is an ancestor of layer i's backward, so the chain-rule
strategy finds control ops right behind the consumer (PAPER §4.3, Alg. 2).

    forward   h[i+1] = matmul(h[i], W[i])            i = 0..L-1, h[0] = x
    backward  g[L]   = neg(h[L])
              d[i]   = mul(g[i+1], h[i+1])            "activation derivative"
              dW[i]  = matmul(h[i], d[i])
              g[i]   = matmul(d[i], W[i])             i = L-1..1
    update    W[i]  <- sub(W[i], dW[i])               update edge into W[i]

A default rewrite swaps h[1..L] (8 tensors at L=8) with two swap-ins each.
Operand order follows the interpreter's rule (ascending origin tensor id).
Inputs: ``numpy.random.default_rng(seed)`` standard normal, weights scaled
by 1/sqrt(N) so values stay O(1) through the chain in fp32.
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

    def node(name, scope, kind=NodeKind.COMPUTE, phase=Phase.UNKNOWN):
        nid = len(nodes)
        param = kind in (NodeKind.VARIABLE, NodeKind.CONSTANT)
        nodes.append(OpNode(nid, name, scope, kind, param, phase, "acc:0", 0.0 if param else 1.0))
        tensors.append(TensorSpec(len(tensors), nid, nbytes, dtype))
        return nid, len(tensors) - 1

    def op(name, scope, phase, *reads):
        nid, tid = node(name, scope, phase=phase)
        for r in reads:
            edges.append(EdgeRec(tensors[r].producer, nid, EdgeAction.READ, r))
        return nid, tid

    _, x = node("x", "input", NodeKind.VARIABLE)
    weights = [node(f"W{i}", f"params/l{i}", NodeKind.VARIABLE) for i in range(layers)]
    h = [x]
    for i in range(layers):
        h.append(op("matmul", f"model/l{i}", Phase.FORWARD, h[i], weights[i][1])[1])
    g = op("neg", "grads/top", Phase.BACKWARD, h[layers])[1]
    for i in reversed(range(layers)):
        d = op("mul", f"grads/l{i}/act", Phase.BACKWARD, g, h[i + 1])[1]
        dw = op("matmul", f"grads/l{i}/dw", Phase.BACKWARD, h[i], d)[1]
        if i > 0:
            g = op("matmul", f"grads/l{i}/dx", Phase.BACKWARD, d, weights[i][1])[1]
        unid, upd = op("sub", f"optimizer/l{i}", Phase.UPDATE, weights[i][1], dw)
        edges.append(EdgeRec(unid, weights[i][0], EdgeAction.UPDATE, upd))
    return CompGraph(nodes, edges, tensors)


def ffchain_inputs(g: CompGraph, n: int, seed: int = 0) -> dict[str, np.ndarray]:
    """float64 N×N per variable, drawn in ascending node id order."""
    rng = np.random.default_rng(seed)
    out = {}
    for nd in g.nodes:
        if nd.parameterized:
            scale = 1.0 if nd.name == "x" else 1.0 / np.sqrt(n)
            out[nd.name] = rng.standard_normal((n, n)) * scale
    return out


# ---------------------------------------------------------------------------
# 3D U-Net (BASELINE config 3): the Çiçek et al. layout the paper trains at
# 192^3.  Built from torch.nn modules; it is a workload
# for the swap path, not part of the path itself.

def unet3d(in_channels: int = 1, classes: int = 2, base: int = 32, depth: int = 3):
    """3D U-Net: per level two (3x3x3 conv, BN, ReLU); 2x max-pool down,
    2x transposed-conv up, skip concatenation; 1x1x1 conv head.  Channels
    base, 2base, ... doubling per level (Çiçek: 32/64 .. 256/512)."""
    import torch
    from torch import nn

    def block(cin, cmid, cout):
        return nn.Sequential(
            nn.Conv3d(cin, cmid, 3, padding=1, bias=False), nn.BatchNorm3d(cmid), nn.ReLU(inplace=True),
            nn.Conv3d(cmid, cout, 3, padding=1, bias=False), nn.BatchNorm3d(cout), nn.ReLU(inplace=True))

    class UNet3D(nn.Module):
        def __init__(self):
            super().__init__()
            self.down = nn.ModuleList()
            self.pool = nn.MaxPool3d(2)
            c = in_channels
            outs = []
            for lvl in range(depth):
                cmid = base * 2 ** lvl
                self.down.append(block(c, cmid, 2 * cmid))
                c = 2 * cmid
                outs.append(c)
            self.bottom = block(c, c, 2 * c)
            c = 2 * c
            self.up = nn.ModuleList()
            self.dec = nn.ModuleList()
            for lvl in reversed(range(depth)):
                self.up.append(nn.ConvTranspose3d(c, c, 2, stride=2))
                skip = outs[lvl]
                self.dec.append(block(c + skip, skip, skip))
                c = skip
            self.head = nn.Conv3d(c, classes, 1)

        def forward(self, x):
            skips = []
            for d in self.down:
                x = d(x)
                skips.append(x)
                x = self.pool(x)
            x = self.bottom(x)
            for up, dec in zip(self.up, self.dec):
                x = up(x)
                x = dec(torch.cat([x, skips.pop()], dim=1))
            return self.head(x)

    return UNet3D()
