"""The transfer/memory model restatement (oracle/sim_oracle.py) vs the reference simulator.

Goldens: reference ``simulate`` reports on generator graphs and seeded
training graphs, plain and rewritten, under four link configurations
(default, serial oracle, slow per-direction links, one shared channel).
Peaks, makespan, transfer time, transfer waits and the full event trace
(hashed) must be identical.
"""

import hashlib
import json
import math

from oracle.sim_oracle import simulate
from paper_1807_02037_b200 import graph_from_dict, topo_order

MIB = 1 << 20
SIMS = {
    "default": dict(),
    "serial": dict(h2d_bw=math.inf, d2h_bw=math.inf, serial=True),
    "slow": dict(h2d_bw=MIB / 1.5, d2h_bw=MIB / 0.75),
    "shared": dict(h2d_bw=float(MIB), d2h_bw=float(MIB), overlap=False),
}


def test_model_matches_reference_simulator(sim_cases):
    for case in sim_cases:
        g = graph_from_dict(case["graph"])
        rep = simulate(g, topo_order(g), **SIMS[case["sim"]])
        trace = rep.pop("event_trace")
        want = dict(case["report"])
        sha = want.pop("trace_sha256")
        n = want.pop("trace_len")
        assert rep == want, (case["name"], case["variant"], case["sim"])
        assert len(trace) == n
        assert hashlib.sha256(json.dumps(trace, sort_keys=True).encode()).hexdigest() == sha, \
            (case["name"], case["variant"], case["sim"])
