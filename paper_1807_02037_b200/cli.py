"""``python -m paper_1807_02037_b200`` — the reference CLI's subcommands (cli.py:45-246).

Same subcommands, flags, file formats, stdout summaries and exit codes as the
reference ``swapgraph`` command, so scripted sweeps switch by changing the
module name:

  generate    synthetic training graph -> canonical JSON (generate.py)
  rewrite     swap insertion + control ops (the drop-in rewrite) -> JSON + report
  simulate    the schedule RUN on the GPU (simulate.py, measured, not modelled):
              the SimReport JSON and its summary; without a CUDA device it
              exits 1 with the error (there is no CPU model to fall back to)
  report      compare two simulation reports
  export-dot  Graphviz DOT of a graph

``SWAPGRAPH_LOG`` = quiet | info | debug sets the log level (cli.py:25-36).
"""

from __future__ import annotations

import argparse
import json
import logging
import os
import sys

from . import serialize
from .generate import TOPOLOGIES
from .graph import topo_order, validate
from .report import DeadlockError, SimConfig
from .rewriter import RewriteConfig, RewriteError, rewrite

_LEVELS = {"quiet": logging.ERROR, "info": logging.INFO, "debug": logging.DEBUG}

# (flag, argparse kwargs, RewriteConfig field or None): one table drives the
# parser and the config, so every RewriteConfig knob has its flag
_SETS = ("optimizer_scopes", "starting_op_names", "excl_scopes", "incl_scopes", "excl_types", "incl_types")
_REWRITE_FLAGS = [
    ("--optimizer-scopes", dict(default="", help="comma-separated scope prefixes of backward/update ops")),
    ("--starting-scope", dict(default=None)),
    ("--starting-op-names", dict(default="")),
    ("--excl-scopes", dict(default="")),
    ("--incl-scopes", dict(default="")),
    ("--excl-types", dict(default="")),
    ("--incl-types", dict(default="")),
    ("--n-tensors", dict(type=int, default=-1)),
    ("--lb", dict(type=int, default=1)),
    ("--ub", dict(type=int, default=10000)),
    ("--ctrld-strategy", dict(choices=["chain_rule", "direct_order"], default="chain_rule")),
    ("--fuse-swapins", dict(action=argparse.BooleanOptionalAction, default=False)),
    ("--swapin-fuse-distance", dict(type=int, default=1)),
    ("--swap-branches", dict(action=argparse.BooleanOptionalAction, default=False)),
    ("--branch-threshold", dict(type=int, default=0)),
]


def _names(raw):
    return frozenset(p.strip() for p in (raw or "").split(",") if p.strip())


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1807_02037_b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="command", required=True)
    g = sub.add_parser("generate", help="emit a synthetic training graph")
    g.add_argument("--topology", choices=sorted(TOPOLOGIES), required=True)
    g.add_argument("--size", type=int, required=True, help="layers / depth / blocks depending on topology")
    g.add_argument("--tensor-bytes", type=int, default=1 << 20)
    g.add_argument("-o", "--output", required=True, help="graph JSON path")
    r = sub.add_parser("rewrite", help="insert swap-out/swap-in pairs")
    r.add_argument("-i", "--input", required=True)
    r.add_argument("-o", "--output", required=True)
    r.add_argument("--report", help="write the rewrite report JSON here")
    for flag, kw in _REWRITE_FLAGS:
        r.add_argument(flag, **kw)
    s = sub.add_parser("simulate", help="run the schedule on the GPU and report what was measured")
    s.add_argument("-i", "--input", required=True)
    s.add_argument("-o", "--output", required=True, help="simulation report JSON path")
    s.add_argument("--device-capacity-bytes", type=int, default=16 * 2**30)
    s.add_argument("--h2d-bandwidth", type=float, default=float(80 * 2**30))
    s.add_argument("--d2h-bandwidth", type=float, default=float(80 * 2**30))
    s.add_argument("--overlap-transfers", action=argparse.BooleanOptionalAction, default=True)
    s.add_argument("--serial", action="store_true", help="single engine, instantaneous transfers (config only)")
    s.add_argument("--trace-csv", help="also write the event trace as CSV")
    s.add_argument("--cost-unit-s", type=float, default=0.0,
                   help="seconds each unit of an op's cost_hint keeps the GPU busy (extension)")
    c = sub.add_parser("report", help="compare two simulation reports")
    c.add_argument("baseline")
    c.add_argument("candidate")
    c.add_argument("--json", action="store_true", help="print the comparison as JSON instead of text")
    d = sub.add_parser("export-dot", help="render a graph to Graphviz DOT")
    d.add_argument("-i", "--input", required=True)
    d.add_argument("-o", "--output", required=True)
    return ap


def _checked(path):
    g = serialize.load_graph(path)
    bad = validate(g)
    if bad:
        raise ValueError(f"{path}: graph is invalid:\n" + "\n".join(f"  {v.code}: {v.message}" for v in bad))
    return g


def _write_json(path, obj):
    with open(path, "w") as fh:
        json.dump(obj, fh, sort_keys=True, indent=2)
        fh.write("\n")


def cmd_generate(a):
    g = TOPOLOGIES[a.topology](a.size, tensor_bytes=a.tensor_bytes)
    serialize.save_graph(g, a.output)
    print(f"wrote {a.topology} graph: {len(g.nodes)} nodes, {len(g.edges)} edges, "
          f"{len(g.tensors)} tensors -> {a.output}")
    return 0


def cmd_rewrite(a):
    g = _checked(a.input)
    kw = {}
    for flag, _ in _REWRITE_FLAGS:
        field = flag[2:].replace("-", "_")
        v = getattr(a, field)
        kw[field] = _names(v) if field in _SETS else v
    out, rep = rewrite(g, RewriteConfig(**kw))
    serialize.save_graph(out, a.output)
    if a.report:
        _write_json(a.report, rep.to_dict())
    for label, v in (("tensors_swapped", rep.tensors_swapped), ("swap_outs", rep.swap_outs_added),
                     ("swap_ins", rep.swap_ins_added), ("control_edges", rep.control_edges_added)):
        print(f"{label}: {v}")
    return 0


def cmd_simulate(a):
    from .simulate import simulate
    g = _checked(a.input)
    if a.serial:
        cfg = SimConfig.serial_oracle(device_capacity_bytes=a.device_capacity_bytes)
    else:
        cfg = SimConfig(device_capacity_bytes=a.device_capacity_bytes, host_to_device_bandwidth=a.h2d_bandwidth,
                        device_to_host_bandwidth=a.d2h_bandwidth, overlap_transfers=a.overlap_transfers)
    rep = simulate(g, topo_order(g), cfg, cost_unit_s=a.cost_unit_s)
    _write_json(a.output, rep.to_dict())
    if a.trace_csv:
        serialize.write_trace_csv(rep.event_trace, a.trace_csv)
    for k in ("peak_device_bytes", "peak_host_bytes", "makespan", "transfer_time_total",
              "transfer_wait_total", "oom"):
        print(f"{k}: {getattr(rep, k)}")
    return 0


def cmd_report(a):
    with open(a.baseline) as fh:
        b = json.load(fh)
    with open(a.candidate) as fh:
        c = json.load(fh)
    cp = c["peak_device_bytes"]
    ratio = b["peak_device_bytes"] / cp if cp else float("inf")
    cmp_ = {"device_peak_baseline": b["peak_device_bytes"], "device_peak_candidate": cp,
            "device_peak_ratio": ratio,
            "host_peak_baseline": b["peak_host_bytes"], "host_peak_candidate": c["peak_host_bytes"],
            "makespan_baseline": b["makespan"], "makespan_candidate": c["makespan"],
            "makespan_overhead": c["makespan"] - b["makespan"],
            "transfer_time_baseline": b["transfer_time_total"], "transfer_time_candidate": c["transfer_time_total"],
            "transfer_wait_baseline": b.get("transfer_wait_total", 0.0),
            "transfer_wait_candidate": c.get("transfer_wait_total", 0.0)}
    if a.json:
        print(json.dumps(cmp_, sort_keys=True, indent=2))
        return 0
    print(f"device peak: {b['peak_device_bytes']} -> {cp} bytes")
    print(f"device_peak_ratio: {ratio:.2f}x")
    print(f"host peak: {b['peak_host_bytes']} -> {c['peak_host_bytes']} bytes")
    print(f"makespan: {b['makespan']} -> {c['makespan']} (overhead {cmp_['makespan_overhead']:+g})")
    print(f"transfer time: {b['transfer_time_total']} -> {c['transfer_time_total']}")
    return 0


def cmd_export_dot(a):
    g = _checked(a.input)
    with open(a.output, "w") as fh:
        fh.write(serialize.to_dot(g, topo_order(g)))
    print(f"wrote DOT for {len(g.nodes)} nodes -> {a.output}")
    return 0


COMMANDS = {"generate": cmd_generate, "rewrite": cmd_rewrite, "simulate": cmd_simulate,
            "report": cmd_report, "export-dot": cmd_export_dot}


def main(argv=None) -> int:
    level = os.environ.get("SWAPGRAPH_LOG", "quiet").lower()
    if level not in _LEVELS:
        print(f"warning: SWAPGRAPH_LOG={level!r} not one of quiet/info/debug", file=sys.stderr)
    logging.basicConfig(level=_LEVELS.get(level, logging.ERROR), stream=sys.stderr,
                        format="%(levelname)s %(name)s: %(message)s")
    a = build_parser().parse_args(argv)
    from .runtime import LmsError
    try:
        return COMMANDS[a.command](a)
    except (serialize.GraphFormatError, RewriteError, DeadlockError, ValueError, OSError, LmsError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
