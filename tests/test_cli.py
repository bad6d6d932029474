"""CLI parity (reference cli.py:45-246 and its tests, tests/test_cli.py): the same
subcommands, flags, stdout summaries and exit codes.  ``simulate`` measures on
the GPU (tests/test_simulate_gpu.py covers it there); here it must fail cleanly."""

import dataclasses
import json

import pytest

from paper_1807_02037_b200 import RewriteConfig, SimConfig, dumps, load_graph, rewrite
from paper_1807_02037_b200.cli import build_parser, main


def cli(capsys, *argv):
    code = main(list(argv))
    cap = capsys.readouterr()
    return code, cap.out, cap.err


def test_pipeline_summaries_match_reference(tmp_path, capsys):
    # the reference's expected stdout for chain(20) (its test_cli.py:23-72)
    g, out_g = tmp_path / "g.json", tmp_path / "swapped.json"
    code, out, _ = cli(capsys, "generate", "--topology", "chain", "--size", "20", "-o", str(g))
    assert code == 0 and out == f"wrote chain graph: 81 nodes, 139 edges, 81 tensors -> {g}\n"
    code, out, _ = cli(capsys, "rewrite", "-i", str(g), "-o", str(out_g))
    assert code == 0
    assert out.splitlines() == ["tensors_swapped: 20", "swap_outs: 20", "swap_ins: 20", "control_edges: 19"]
    assert out_g.read_text() == dumps(rewrite(load_graph(str(g)), RewriteConfig())[0])
    # report over the reference model's two reports for that pipeline
    base = dict(peak_device_bytes=22020096, peak_host_bytes=0, makespan=60.0, transfer_time_total=0.0,
                transfer_wait_total=0.0, oom=False, event_trace=[])
    cand = dict(peak_device_bytes=3145728, peak_host_bytes=20971520, makespan=60.0000244140625,
                transfer_time_total=0.0004882812500000002, transfer_wait_total=0.0, oom=False, event_trace=[])
    (tmp_path / "b.json").write_text(json.dumps(base))
    (tmp_path / "c.json").write_text(json.dumps(cand))
    code, out, _ = cli(capsys, "report", str(tmp_path / "b.json"), str(tmp_path / "c.json"))
    assert code == 0
    assert out.splitlines() == [
        "device peak: 22020096 -> 3145728 bytes",
        "device_peak_ratio: 7.00x",
        "host peak: 0 -> 20971520 bytes",
        "makespan: 60.0 -> 60.0000244140625 (overhead +2.44141e-05)",
        "transfer time: 0.0 -> 0.0004882812500000002",
    ]
    code, out, _ = cli(capsys, "report", str(tmp_path / "b.json"), str(tmp_path / "c.json"), "--json")
    doc = json.loads(out)
    assert doc["device_peak_ratio"] == 7.0 and doc["makespan_overhead"] == pytest.approx(2.44140625e-05)


def test_rewrite_report_and_cap_zero(tmp_path, capsys):
    g = tmp_path / "g.json"
    cli(capsys, "generate", "--topology", "chain", "--size", "5", "-o", str(g))
    rep = tmp_path / "r.json"
    code, _, _ = cli(capsys, "rewrite", "-i", str(g), "-o", str(tmp_path / "o.json"), "--report", str(rep))
    assert code == 0 and json.loads(rep.read_text())["tensors_swapped"] == 5
    same = tmp_path / "same.json"
    code, _, _ = cli(capsys, "rewrite", "-i", str(g), "-o", str(same), "--n-tensors", "0")
    assert code == 0 and same.read_text() == dumps(load_graph(str(g)))


def test_export_dot(tmp_path, capsys):
    g = tmp_path / "g.json"
    cli(capsys, "generate", "--topology", "branchy", "--size", "4", "-o", str(g))
    d = tmp_path / "g.dot"
    code, out, _ = cli(capsys, "export-dot", "-i", str(g), "-o", str(d))
    assert code == 0 and d.read_text().startswith("digraph g {") and "style=dashed" not in d.read_text()
    assert out.endswith(f"-> {d}\n")


def test_parser_exposes_every_config_field_with_its_default():
    args = build_parser().parse_args(["rewrite", "-i", "a", "-o", "b"])
    cfg = RewriteConfig()
    for f in dataclasses.fields(RewriteConfig):
        assert f.name in vars(args), f.name
        if not isinstance(getattr(cfg, f.name), frozenset):
            assert getattr(args, f.name) == getattr(cfg, f.name), f.name
    sim = build_parser().parse_args(["simulate", "-i", "a", "-o", "b"])
    sc = SimConfig()
    assert (sim.device_capacity_bytes, sim.h2d_bandwidth, sim.d2h_bandwidth, sim.overlap_transfers) == (
        sc.device_capacity_bytes, sc.host_to_device_bandwidth, sc.device_to_host_bandwidth, sc.overlap_transfers)
    p = build_parser()
    assert p.parse_args(["rewrite", "-i", "a", "-o", "b", "--fuse-swapins"]).fuse_swapins
    assert not p.parse_args(["rewrite", "-i", "a", "-o", "b", "--no-fuse-swapins"]).fuse_swapins
    assert not p.parse_args(["simulate", "-i", "a", "-o", "b", "--no-overlap-transfers"]).overlap_transfers


def test_failures_exit_one_with_error(tmp_path, capsys):
    code, out, err = cli(capsys, "rewrite", "-i", str(tmp_path / "nope.json"), "-o", str(tmp_path / "o.json"))
    assert code == 1 and out == "" and err.startswith("error: ")
    bad = tmp_path / "bad.json"
    bad.write_text("{ not json")
    code, _, err = cli(capsys, "export-dot", "-i", str(bad), "-o", str(tmp_path / "x.dot"))
    assert code == 1 and err.startswith(f"error: {bad}: line 1")
    doc = {"nodes": [{"id": 0, "name": "x", "kind": "variable", "parameterized": True, "device": "acc:0"},
                     {"id": 1, "name": "f", "kind": "compute", "parameterized": False, "device": "acc:0"}],
           "edges": [{"src": 0, "dst": 1, "action": "read", "tensor": 7}],
           "tensors": [{"id": 0, "producer": 0, "size_bytes": 8}]}
    inv = tmp_path / "invalid.json"
    inv.write_text(json.dumps(doc))
    code, _, err = cli(capsys, "export-dot", "-i", str(inv), "-o", str(tmp_path / "g.dot"))
    assert code == 1 and "graph is invalid" in err and "unknown-tensor" in err
    g = tmp_path / "g.json"
    cli(capsys, "generate", "--topology", "chain", "--size", "3", "-o", str(g))
    code, _, err = cli(capsys, "rewrite", "-i", str(g), "-o", str(tmp_path / "o.json"), "--lb", "0")
    assert code == 1 and "error: lb must be positive" in err
    with pytest.raises(SystemExit) as exc:
        main(["generate", "--topology", "hourglass", "--size", "3", "-o", str(tmp_path / "h.json")])
    assert exc.value.code == 2


def test_simulate_without_gpu_fails_cleanly(tmp_path, capsys):
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check (tests/test_cli_gpu.py runs it on the GPU)")
    g = tmp_path / "g.json"
    cli(capsys, "generate", "--topology", "chain", "--size", "3", "-o", str(g))
    code, out, err = cli(capsys, "simulate", "-i", str(g), "-o", str(tmp_path / "r.json"))
    assert code == 1 and out == "" and "CUDA" in err


def test_log_level_warning(tmp_path, capsys, monkeypatch):
    monkeypatch.setenv("SWAPGRAPH_LOG", "loud")
    code, _, err = cli(capsys, "generate", "--topology", "chain", "--size", "3", "-o", str(tmp_path / "g.json"))
    assert code == 0 and "warning: SWAPGRAPH_LOG='loud'" in err
