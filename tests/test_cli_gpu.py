"""The CLI's ``simulate`` on the GPU: the measured report file has the reference
schema (sim.py:84-113) and, for the plain chain(20), the reference model's
device peak (its test_cli.py:43-53: 22020096 bytes)."""

import json

import pytest

from paper_1807_02037_b200.cli import main

pytestmark = pytest.mark.gpu


def test_cli_simulate_measures(tmp_path, capsys, lms_ctx):
    g, sw = tmp_path / "g.json", tmp_path / "s.json"
    assert main(["generate", "--topology", "chain", "--size", "20", "-o", str(g)]) == 0
    assert main(["rewrite", "-i", str(g), "-o", str(sw)]) == 0
    capsys.readouterr()
    assert main(["simulate", "-i", str(g), "-o", str(tmp_path / "b.json"), "--serial"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == "peak_device_bytes: 22020096" and out[5] == "oom: False"
    csv = tmp_path / "t.csv"
    assert main(["simulate", "-i", str(sw), "-o", str(tmp_path / "c.json"), "--trace-csv", str(csv)]) == 0
    rep = json.loads((tmp_path / "c.json").read_text())
    assert set(rep) == {"peak_device_bytes", "peak_host_bytes", "makespan", "transfer_time_total",
                        "transfer_wait_total", "oom", "event_trace"}
    assert rep["peak_host_bytes"] > 0 and rep["transfer_time_total"] > 0
    assert csv.read_text().startswith("time,event,node,tensor,bytes")
    assert main(["report", str(tmp_path / "b.json"), str(tmp_path / "c.json")]) == 0
