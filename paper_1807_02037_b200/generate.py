"""Deterministic synthetic training-step graphs (chain, branchy, unet, resnet_like).

Same graphs, ids included, as ``swapgraph/generate.py:88-210`` (pinned by
``tests/golden``): a forward stack whose activations are re-read by a
mirrored backward chain, plus one update op per weight variable.
Activations/gradients are ``tensor_bytes``; weights are 64 bytes.
"""

from __future__ import annotations

from .graph import CompGraph, EdgeAction, EdgeRec, NodeKind, OpNode, Phase, TensorSpec

PARAM_BYTES = 64


class _Step:
    """Append-only builder: node ids and tensor ids are positions."""

    def __init__(self, device: str = "acc:0"):
        self.device = device
        self.nodes: list[OpNode] = []
        self.edges: list[EdgeRec] = []
        self.tensors: list[TensorSpec] = []
        self.var_tensor: dict[int, int] = {}

    def _new(self, node: OpNode, out_bytes: int) -> int:
        self.nodes.append(node)
        tid = len(self.tensors)
        self.tensors.append(TensorSpec(tid, node.id, out_bytes))
        return tid

    def var(self, name: str, nbytes: int) -> tuple[int, int]:
        nid = len(self.nodes)
        tid = self._new(OpNode(nid, name, "params", NodeKind.VARIABLE, True, Phase.UNKNOWN,
                               self.device, 0.0), nbytes)
        self.var_tensor[nid] = tid
        return nid, tid

    def op(self, name: str, scope: str, phase: Phase, reads, nbytes: int) -> int:
        nid = len(self.nodes)
        for tid in reads:
            self.edges.append(EdgeRec(self.tensors[tid].producer, nid, EdgeAction.READ, tid))
        return self._new(OpNode(nid, name, scope, NodeKind.COMPUTE, False, phase,
                                self.device, 1.0), nbytes)

    def backward_and_updates(self, acts: list[int], weights: list[tuple[int, int]],
                             nbytes: int) -> CompGraph:
        """Mirror ``acts`` backward (each step reads its activation and the
        previous gradient), then one update per (weight var, position)."""
        grad_at: dict[int, int] = {}
        prev = None
        for pos in reversed(range(len(acts))):
            reads = [acts[pos]] if prev is None else [acts[pos], prev]
            prev = grad_at[pos] = self.op(f"bwd_{pos}", f"grads/layer_{pos}",
                                          Phase.BACKWARD, reads, nbytes)
        for var_id, pos in weights:
            upd = self.op(f"upd_{pos}", f"optimizer/layer_{pos}", Phase.UPDATE,
                          [grad_at[pos], self.var_tensor[var_id]], PARAM_BYTES)
            self.edges.append(EdgeRec(self.tensors[upd].producer, var_id, EdgeAction.UPDATE, upd))
        return CompGraph(self.nodes, self.edges, self.tensors)


def _layered(n: int, tensor_bytes: int, skip_every_third: bool) -> CompGraph:
    b = _Step()
    _, act = b.var("x_in", tensor_bytes)
    acts, weights = [], []
    for i in range(n):
        w, wt = b.var(f"w_{i}", PARAM_BYTES)
        reads = [act, wt]
        if skip_every_third and i >= 4 and (i - 4) % 3 == 0:
            reads.append(acts[i - 4])
        act = b.op(f"fwd_{i}", f"model/layer_{i}", Phase.FORWARD, reads, tensor_bytes)
        acts.append(act)
        weights.append((w, i))
    return b.backward_and_updates(acts, weights, tensor_bytes)


def chain(n: int, tensor_bytes: int = 1 << 20) -> CompGraph:
    """``n`` forward layers, each activation re-read by its backward op."""
    if n < 1:
        raise ValueError("chain needs at least one layer")
    return _layered(n, tensor_bytes, skip_every_third=False)


def branchy(n: int, tensor_bytes: int = 1 << 20) -> CompGraph:
    """Chain plus a skip edge from layer i-4 into layers 4, 7, 10, ..."""
    if n < 2:
        raise ValueError("branchy needs at least two layers")
    return _layered(n, tensor_bytes, skip_every_third=True)


def unet(depth: int, tensor_bytes: int = 1 << 20) -> CompGraph:
    """Encoder/decoder with a long skip edge per level."""
    if depth < 1:
        raise ValueError("unet needs depth >= 1")
    b = _Step()
    _, act = b.var("x_in", tensor_bytes)
    acts, weights = [], []

    def level(prefix: str, extra: list[int]) -> int:
        nonlocal act
        pos = len(acts)
        w, wt = b.var(f"w_{pos}", PARAM_BYTES)
        act = b.op(f"{prefix}_{pos}", f"model/{prefix}_{pos}", Phase.FORWARD,
                   [act] + extra + [wt], tensor_bytes)
        acts.append(act)
        weights.append((w, pos))
        return act

    skips = [level("enc", []) for _ in range(depth)]
    level("mid", [])
    for j in reversed(range(depth)):
        level("dec", [skips[j]])
    return b.backward_and_updates(acts, weights, tensor_bytes)


def resnet_like(blocks: int, tensor_bytes: int = 1 << 20) -> CompGraph:
    """Stem plus ``blocks`` residual blocks (two convs and a join each)."""
    if blocks < 1:
        raise ValueError("resnet_like needs at least one block")
    b = _Step()
    _, x = b.var("x_in", tensor_bytes)
    w, wt = b.var("w_stem", PARAM_BYTES)
    r = b.op("stem", "model/stem", Phase.FORWARD, [x, wt], tensor_bytes)
    outs, weights = [r], [(w, 0)]
    for k in range(1, blocks + 1):
        w1, w1t = b.var(f"w_{k}a", PARAM_BYTES)
        t1 = b.op(f"conv_{k}a", f"model/block_{k}", Phase.FORWARD, [r, w1t], tensor_bytes)
        _, w2t = b.var(f"w_{k}b", PARAM_BYTES)
        t2 = b.op(f"conv_{k}b", f"model/block_{k}", Phase.FORWARD, [t1, w2t], tensor_bytes)
        r = b.op(f"join_{k}", f"model/block_{k}", Phase.FORWARD, [t2, r], tensor_bytes)
        outs.append(r)
        weights.append((w1, k))
    return b.backward_and_updates(outs, weights, tensor_bytes)


TOPOLOGIES = {"chain": chain, "branchy": branchy, "unet": unet, "resnet_like": resnet_like}
