"""Generate golden vectors by running the REFERENCE implementation (swapgraph).

Run in the build container, where the read-only reference exists:

    python tests/golden/make_golden.py

It imports ``swapgraph`` from /root/reference/pkg/src and the reference's
own test fixtures/graph generators from /root/reference/pkg/tests, and
writes small gzipped JSON files next to this script:

* ``rewrite_cases.json.gz``   input graphs x config grid -> sha256 of the
                              reference ``dumps(rewrite(g, cfg))`` + the
                              report dict (or the error message); full text
                              for a few named cases
* ``ctrl_queries.json.gz``    criterion-3 query set (test_acceptance.py:99-139)
                              -> reference direct_order / chain_rule answers
* ``interp_cases.json.gz``    interpret() inputs and outputs (float64, exact
                              repr) for graphgen seeds and the C1 ffchain,
                              before and after rewrite
* ``sim_cases.json.gz``       simulate() reports (no trace) for the memory /
                              transfer model restatement in oracle/

Nothing at test time reads /root/reference; the tests only read these files.
"""

from __future__ import annotations

import gzip
import hashlib
import itertools
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import swapgraph as R  # noqa: E402  (the reference)
import fixtures as F  # noqa: E402
import graphgen  # noqa: E402
from swapgraph import generate as RG  # noqa: E402
from swapgraph.control import CtrlQuery  # noqa: E402

from paper_1807_02037_b200 import workloads  # noqa: E402
from paper_1807_02037_b200.serialize import graph_to_dict as our_to_dict  # noqa: E402

MIB = 1 << 20


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def cfg_dict(cfg: R.RewriteConfig) -> dict:
    d = {}
    for k, v in cfg.__dict__.items():
        d[k] = sorted(v) if isinstance(v, frozenset) else v
    return d


def source_graphs():
    out = []
    for name in ("expression_graph", "variable_refresh_graph", "hot_fanout_graph",
                 "order_chain_graph", "two_layer_training_graph", "three_op_chain",
                 "clustered_consumers_graph", "training_expression_graph"):
        out.append((f"fixture:{name}", getattr(F, name)()))
    out.append(("fixture:replay_chain(30)", F.replay_chain(30, tensor_bytes=MIB)))
    for n in (1, 3, 12, 20, 100):
        out.append((f"gen:chain({n})", RG.chain(n)))
    out += [("gen:branchy(8)", RG.branchy(8)), ("gen:branchy(20)", RG.branchy(20)),
            ("gen:unet(3)", RG.unet(3)), ("gen:unet(4,8MiB)", RG.unet(4, tensor_bytes=8 * MIB)),
            ("gen:resnet_like(4)", RG.resnet_like(4)), ("gen:resnet_like(16)", RG.resnet_like(16))]
    for seed in range(200):
        out.append((f"graphgen:{seed}", graphgen.training_graph(seed)))
    for L in (1, 3, 8):
        g = R.graph_from_dict(our_to_dict(workloads.ffchain(L, 16)))
        out.append((f"ffchain({L},16)", g))
    return out


def config_grid():
    grid = [R.RewriteConfig(n_tensors=n, lb=lb, ctrld_strategy=s, fuse_swapins=f)
            for n, lb, s, f in itertools.product((0, 3, -1), (1, 3), ("chain_rule", "direct_order"),
                                                 (False, True))]
    grid += [
        R.RewriteConfig(lb=1, ub=3),
        R.RewriteConfig(lb=2, ub=4, ctrld_strategy="direct_order"),
        R.RewriteConfig(lb=5, ub=9, ctrld_strategy="direct_order", swap_branches=True,
                        branch_threshold=5),
        R.RewriteConfig(swap_branches=True, branch_threshold=1, ctrld_strategy="direct_order"),
        R.RewriteConfig(swap_branches=True, branch_threshold=4, fuse_swapins=True,
                        swapin_fuse_distance=3),
        R.RewriteConfig(fuse_swapins=True, swapin_fuse_distance=0),
        R.RewriteConfig(fuse_swapins=True, swapin_fuse_distance=7, lb=2),
        R.RewriteConfig(excl_scopes=frozenset({"model/l1", "model/layer_2"})),
        R.RewriteConfig(incl_types=frozenset({"neg"}), excl_types=frozenset({"matmul"})),
        R.RewriteConfig(incl_scopes=frozenset({"grads"}), n_tensors=5),
        R.RewriteConfig(optimizer_scopes=frozenset({"grads", "optimizer"})),
        R.RewriteConfig(starting_scope="model", lb=2),
        R.RewriteConfig(starting_op_names=frozenset({"x", "x_in"})),
        R.RewriteConfig(n_tensors=1, ctrld_strategy="direct_order", ub=2),
    ]
    return grid


def make_rewrite_cases():
    cases = []
    full_text_for = {"fixture:hot_fanout_graph", "gen:chain(20)", "fixture:clustered_consumers_graph",
                     "ffchain(8,16)", "graphgen:7"}
    grid = config_grid()
    for name, g in source_graphs():
        results = []
        for cfg in grid:
            entry = {"cfg": cfg_dict(cfg)}
            try:
                out, rep = R.rewrite(g, cfg)
                text = R.dumps(out)
                entry["sha256"] = sha(text)
                entry["report"] = rep.to_dict()
                if name in full_text_for:
                    entry["dumps"] = text
            except Exception as exc:  # the error text is part of the contract
                entry["error"] = f"{type(exc).__name__}: {exc}"
            results.append(entry)
        cases.append({"name": name, "graph": R.graph_to_dict(g), "input_dumps_sha256": sha(R.dumps(g)),
                      "order": {str(k): v for k, v in R.topo_order(g).items()},
                      "results": results})
    # larger generator cases with the default config only (rewrite planning scale)
    for name, g in (("gen:chain(317)", RG.chain(317)), ("gen:resnet_like(50)", RG.resnet_like(50))):
        out, rep = R.rewrite(g, R.RewriteConfig())
        cases.append({"name": name, "graph": R.graph_to_dict(g), "input_dumps_sha256": sha(R.dumps(g)),
                      "results": [{"cfg": cfg_dict(R.RewriteConfig()), "sha256": sha(R.dumps(out)),
                                   "report": rep.to_dict()}]})
    return cases


def make_ctrl_queries():
    rewritten_chain3, _ = R.rewrite(RG.chain(3), R.RewriteConfig())
    graphs = [("order_chain", F.order_chain_graph()), ("two_layer", F.two_layer_training_graph()),
              ("expression", F.expression_graph()), ("training_expression", F.training_expression_graph()),
              ("clustered", F.clustered_consumers_graph()), ("chain3", RG.chain(3)),
              ("chain3_rewritten", rewritten_chain3)]
    graphs += [(f"graphgen:{s}", graphgen.training_graph(s)) for s in range(10)]
    out = []
    for name, g in graphs:
        order = R.topo_order(g)
        ids = sorted(g.node_by_id)
        answers = []
        for source, target in itertools.permutations(ids, 2):
            if order[source] >= order[target]:
                continue
            for lb in (1, 2, 3, 5):
                for ub in (lb, lb + 2, 10):
                    q = CtrlQuery(source=source, target=target, lb=lb, ub=ub)
                    answers.append([source, target, lb, ub, R.direct_order(g, order, q),
                                    R.chain_rule(g, order, q)])
        fb = []
        for source, target in itertools.permutations(ids, 2):
            fb.append([source, target, R.fallback_control(g, order, source, target)])
        out.append({"name": name, "graph": R.graph_to_dict(g), "queries": answers, "fallback": fb})
    return out


def _arrays(d):
    return {k: np.asarray(v, dtype=np.float64).tolist() for k, v in d.items()}


def make_interp_cases():
    cases = []
    cfgs = [R.RewriteConfig(), R.RewriteConfig(lb=1, ub=3),
            R.RewriteConfig(ctrld_strategy="direct_order", fuse_swapins=True, lb=3)]
    for seed in range(40):
        g = graphgen.training_graph(seed)
        inputs = graphgen.random_inputs(g, seed)
        base = R.interpret(g, inputs)
        rewritten = []
        for cfg in cfgs:
            out, _ = R.rewrite(g, cfg)
            after = R.interpret(out, inputs)
            rewritten.append({"cfg": cfg_dict(cfg), "graph": R.graph_to_dict(out), "outputs": _arrays(after)})
        cases.append({"name": f"graphgen:{seed}", "graph": R.graph_to_dict(g), "inputs": _arrays(inputs),
                      "outputs": _arrays(base), "rewritten": rewritten})
    for L, N in ((3, 8), (8, 16)):
        g = R.graph_from_dict(our_to_dict(workloads.ffchain(L, N)))
        inputs = workloads.ffchain_inputs(workloads.ffchain(L, N), N, seed=0)
        base = R.interpret(g, inputs)
        out, rep = R.rewrite(g, R.RewriteConfig(lb=1, ub=3))
        after = R.interpret(out, inputs)
        cases.append({"name": f"ffchain({L},{N})", "graph": R.graph_to_dict(g), "inputs": _arrays(inputs),
                      "outputs": _arrays(base),
                      "rewritten": [{"cfg": cfg_dict(R.RewriteConfig(lb=1, ub=3)),
                                     "graph": R.graph_to_dict(out), "outputs": _arrays(after),
                                     "report": rep.to_dict()}]})
    return cases


def make_sim_cases():
    cases = []
    sims = [("default", R.SimConfig()), ("serial", R.SimConfig.serial_oracle()),
            ("slow", R.SimConfig(host_to_device_bandwidth=MIB / 1.5, device_to_host_bandwidth=MIB / 0.75)),
            ("shared", R.SimConfig(host_to_device_bandwidth=MIB, device_to_host_bandwidth=MIB,
                                   overlap_transfers=False))]
    graphs = [("gen:chain(20)", RG.chain(20)), ("gen:unet(4,8MiB)", RG.unet(4, tensor_bytes=8 * MIB)),
              ("fixture:replay_chain(30)", F.replay_chain(30, tensor_bytes=MIB)),
              ("gen:resnet_like(6)", RG.resnet_like(6))]
    graphs += [(f"graphgen:{s}", graphgen.training_graph(s, tensor_bytes=64)) for s in range(1000, 1030)]
    for name, g in graphs:
        variants = [("plain", g)]
        for tag, cfg in (("default", R.RewriteConfig()),
                         ("direct_lb2", R.RewriteConfig(lb=2, ctrld_strategy="direct_order")),
                         ("branches", R.RewriteConfig(lb=1, swap_branches=True, branch_threshold=1,
                                                      ctrld_strategy="direct_order", fuse_swapins=True))):
            try:
                variants.append((tag, R.rewrite(g, cfg)[0]))
            except Exception:
                pass
        for vtag, vg in variants:
            order = R.topo_order(vg)
            for stag, scfg in sims:
                rep = R.simulate(vg, order, scfg)
                d = rep.to_dict()
                trace = d.pop("event_trace")
                d["trace_sha256"] = sha(json.dumps(trace, sort_keys=True))
                d["trace_len"] = len(trace)
                cases.append({"name": name, "variant": vtag, "sim": stag, "graph": R.graph_to_dict(vg),
                              "report": d})
    return cases


def write(name, obj):
    path = os.path.join(HERE, name)
    with gzip.open(path, "wt") as fh:
        json.dump(obj, fh, separators=(",", ":"), sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def make_api_cases():
    """The public pass functions on their own (insert_swap_pair, attach_control,
    free_step_oracle) and the reference's import surface (__init__.py:60-115)."""
    graphs = [(f"fixture:{n}", getattr(F, n)()) for n in
              ("expression_graph", "hot_fanout_graph", "three_op_chain", "two_layer_training_graph",
               "clustered_consumers_graph", "training_expression_graph")]
    graphs += [("gen:chain(6)", RG.chain(6)), ("gen:unet(3)", RG.unet(3)), ("gen:resnet_like(3)", RG.resnet_like(3))]
    graphs += [(f"graphgen:{s}", graphgen.training_graph(s)) for s in range(12)]
    inserts, attaches, frees, bares = [], [], [], {}
    for name, g in graphs:
        order = R.topo_order(g)
        cands = R.select_candidates(g, order, R.RewriteConfig(swap_branches=True, branch_threshold=0))
        probes = [e for e, _ in cands][:6]
        probes.append(R.EdgeRec(g.max_node_id() + 5, g.max_node_id() + 6, R.EdgeAction.READ, 0))
        probes += [e for e in g.edges if e.action is not R.EdgeAction.READ][:1]
        for e in probes:
            entry = {"edge": [e.src, e.dst, e.action.value, e.tensor]}
            try:
                out, so, si = R.insert_swap_pair(g, e)
                entry.update(sha256=sha(R.dumps(out)), so=so, si=si)
            except Exception as exc:
                entry["error"] = f"{type(exc).__name__}: {exc}"
            inserts.append(dict(entry, graph=name))
        try:
            out, _ = R.rewrite(g, R.RewriteConfig(n_tensors=2))
        except R.RewriteError:
            out = g   # no phase tags: attach_control still applies to the bare graph
        # drop the rewrite's own control edges so attach_control sees bare swap-ins
        bare = R.CompGraph(out.nodes, tuple(e for e in out.edges if e.action is not R.EdgeAction.CONTROL),
                           out.tensors)
        bares[name + ":bare"] = R.graph_to_dict(bare)
        sis = [n.id for n in bare.nodes if n.kind is R.NodeKind.SWAP_IN][:2]
        ids = sorted(bare.node_by_id)
        for si in sis + [ids[0]]:
            for ctrl in ids[:: max(1, len(ids) // 9)] + [10 ** 6]:
                entry = {"graph": name + ":bare", "ctrl": ctrl, "swap_in": si}
                try:
                    entry["sha256"] = sha(R.dumps(R.attach_control(bare, ctrl, si)))
                except Exception as exc:
                    entry["error"] = f"{type(exc).__name__}: {exc}"
                attaches.append(entry)
        for vg in (g, out):
            vo = R.topo_order(vg)
            frees.append({"graph": R.graph_to_dict(vg), "order": {str(k): v for k, v in vo.items()},
                          "free_steps": {str(t.id): R.free_step_oracle(vg, vo, t.id) for t in vg.tensors}})
    graph_dicts = {name: R.graph_to_dict(g) for name, g in graphs}
    graph_dicts.update(bares)
    return {"reference_all": sorted(R.__all__), "graphs": graph_dicts, "insert_swap_pair": inserts,
            "attach_control": attaches, "free_step_oracle": frees}


if __name__ == "__main__":
    only = sys.argv[1:]
    makers = {"rewrite_cases.json.gz": make_rewrite_cases, "ctrl_queries.json.gz": make_ctrl_queries,
              "interp_cases.json.gz": make_interp_cases, "sim_cases.json.gz": make_sim_cases,
              "api_cases.json.gz": make_api_cases}
    for fname, fn in makers.items():
        if not only or fname in only:
            write(fname, fn())
