"""Wire formats: canonical JSON, Graphviz DOT and trace CSV.

The JSON layout is the reference's (``swapgraph/serialize.py:26-59``):
top-level ``nodes``/``edges``/``tensors`` arrays, sorted, keys sorted,
2-space indent, trailing newline — so ``dumps`` of equal graphs is
byte-identical across the two implementations and the parity tests compare
bytes.  The loader is strict and names the offending field
(serialize.py:62-115).  DOT and CSV follow serialize.py:151-193.
"""

from __future__ import annotations

import csv
import json
from typing import Any

from .graph import CompGraph, EdgeAction, EdgeRec, NodeKind, OpNode, Phase, TensorSpec, edge_sort_key

_NODE_FIELDS = ("id", "name", "scope", "kind", "parameterized", "phase", "device", "cost_hint")


def _node_doc(n: OpNode) -> dict[str, Any]:
    doc = {f: getattr(n, f) for f in _NODE_FIELDS}
    doc["kind"] = n.kind.value
    doc["phase"] = n.phase.value
    return doc


def _edge_doc(e: EdgeRec) -> dict[str, Any]:
    return {"src": e.src, "dst": e.dst, "action": e.action.value, "tensor": e.tensor}


def _tensor_doc(t: TensorSpec) -> dict[str, Any]:
    return {"id": t.id, "producer": t.producer, "size_bytes": t.size_bytes, "dtype": t.dtype}


def graph_to_dict(g: CompGraph) -> dict[str, Any]:
    return {
        "nodes": [_node_doc(n) for n in sorted(g.nodes, key=lambda n: n.id)],
        "edges": [_edge_doc(e) for e in sorted(g.edges, key=edge_sort_key)],
        "tensors": [_tensor_doc(t) for t in sorted(g.tensors, key=lambda t: t.id)],
    }


class GraphFormatError(ValueError):
    """Malformed graph document; the message carries the field context."""


def _field(obj: dict, name: str, where: str):
    try:
        return obj[name]
    except KeyError:
        raise GraphFormatError(f"{where}: missing field {name!r}") from None


def _as_enum(enum_cls, raw, where: str):
    try:
        return enum_cls(raw)
    except ValueError:
        choices = ", ".join(m.value for m in enum_cls)
        raise GraphFormatError(f"{where}: {raw!r} is not one of {choices}") from None


def _parse_node(raw: dict, where: str) -> OpNode:
    return OpNode(
        id=int(_field(raw, "id", where)),
        name=str(_field(raw, "name", where)),
        scope=str(raw.get("scope", "")),
        kind=_as_enum(NodeKind, _field(raw, "kind", where), where),
        parameterized=bool(_field(raw, "parameterized", where)),
        phase=_as_enum(Phase, raw.get("phase", "unknown"), where),
        device=str(_field(raw, "device", where)),
        cost_hint=float(raw.get("cost_hint", 1.0)),
    )


def _parse_edge(raw: dict, where: str) -> EdgeRec:
    tensor = _field(raw, "tensor", where)
    return EdgeRec(
        src=int(_field(raw, "src", where)),
        dst=int(_field(raw, "dst", where)),
        action=_as_enum(EdgeAction, _field(raw, "action", where), where),
        tensor=None if tensor is None else int(tensor),
    )


def _parse_tensor(raw: dict, where: str) -> TensorSpec:
    return TensorSpec(
        id=int(_field(raw, "id", where)),
        producer=int(_field(raw, "producer", where)),
        size_bytes=int(_field(raw, "size_bytes", where)),
        dtype=str(raw.get("dtype", "f32")),
    )


def graph_from_dict(doc: dict[str, Any]) -> CompGraph:
    if not isinstance(doc, dict):
        raise GraphFormatError("top level: expected an object")
    parts = []
    for key, parse in (("nodes", _parse_node), ("edges", _parse_edge), ("tensors", _parse_tensor)):
        parts.append([parse(raw, f"{key}[{i}]")
                      for i, raw in enumerate(_field(doc, key, "top level"))])
    return CompGraph(*parts)


def dumps(g: CompGraph) -> str:
    """Canonical JSON text (sorted keys, indent 2, trailing newline)."""
    return json.dumps(graph_to_dict(g), sort_keys=True, indent=2) + "\n"


def loads(text: str) -> CompGraph:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise GraphFormatError(f"line {exc.lineno}, column {exc.colno}: {exc.msg}") from exc
    return graph_from_dict(doc)


def save_graph(g: CompGraph, path: str) -> None:
    with open(path, "w") as fh:
        fh.write(dumps(g))


def load_graph(path: str) -> CompGraph:
    with open(path) as fh:
        text = fh.read()
    try:
        return loads(text)
    except GraphFormatError as exc:
        raise GraphFormatError(f"{path}: {exc}") from None


_STYLE = {EdgeAction.READ: "solid", EdgeAction.UPDATE: "dotted", EdgeAction.CONTROL: "dashed"}


def to_dot(g: CompGraph, order: dict[int, int] | None = None) -> str:
    """Graphviz DOT: one cluster per device; read solid, update dotted,
    control dashed; parameterized nodes double-circled."""
    clusters: dict[str, list[OpNode]] = {}
    for n in g.nodes:
        clusters.setdefault(n.device, []).append(n)
    out = ["digraph g {", "  rankdir=TB;"]
    for i, dev in enumerate(sorted(clusters)):
        out += [f"  subgraph cluster_{i} {{", f'    label="{dev}";']
        for n in clusters[dev]:
            label = n.name
            if order is not None and n.id in order:
                label += f"\\n{order[n.id]}"
            shape = "doublecircle" if n.parameterized else "circle"
            out.append(f'    n{n.id} [label="{label}" shape={shape}];')
        out.append("  }")
    for e in sorted(g.edges, key=edge_sort_key):
        attrs = "style=" + _STYLE[e.action]
        if e.tensor is not None:
            attrs += f' label="t{e.tensor}"'
        out.append(f"  n{e.src} -> n{e.dst} [{attrs}];")
    out.append("}")
    return "\n".join(out) + "\n"


def write_trace_csv(events, path: str) -> None:
    """Trace rows ``time,event,node,tensor,bytes`` (serialize.py:181-193).

    Accepts simulator ``TraceEvent``s and the executor's measured events
    alike, so measured and modelled timelines diff directly.
    """
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["time", "event", "node", "tensor", "bytes"])
        for ev in events:
            w.writerow([ev.time, ev.event, "" if ev.node is None else ev.node,
                        "" if ev.tensor is None else ev.tensor, ev.bytes])
