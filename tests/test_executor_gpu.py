"""GPU executor parity (SURVEY §8(c) rules 2 and 3).

* swap vs no-swap on the GPU: bit-equal (swapping is a copy);
* GPU (fp32) vs the fp64 oracle interpreter: relative error within fp32
  tolerance; GPU in fp64 vs oracle: 1e-12;
* the measured report: swap traffic happened and the pool's peak drops
  when tensors are swapped.
"""

import numpy as np
import pytest
import torch

from oracle.interp_oracle import interpret as oracle_interpret
from paper_1807_02037_b200 import RewriteConfig, graph_from_dict, rewrite
from paper_1807_02037_b200.executor import ExecConfig, execute
from paper_1807_02037_b200.workloads import ffchain, ffchain_inputs

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("codec", ["ce", "sm", "zvc"])
def test_golden_graphs_fp64_match_oracle(lms_ctx, interp_cases, codec):
    for case in interp_cases:
        inputs = {k: np.asarray(v) for k, v in case["inputs"].items()}
        want = {k: np.asarray(v) for k, v in case["outputs"].items()}
        for rw in case["rewritten"]:
            g = graph_from_dict(rw["graph"])
            got, rep = execute(g, inputs, ExecConfig(dtype="float64", codec=codec), ctx=lms_ctx)
            for k in want:
                assert np.allclose(got[k], want[k], rtol=1e-12, atol=1e-12), (case["name"], k)


@pytest.mark.parametrize("L,N", [(8, 256), (8, 1024)])
def test_ffchain_swap_equals_noswap_and_oracle(lms_ctx, L, N):
    g = ffchain(L, N)
    inputs = ffchain_inputs(g, N, seed=0)
    base, rep0 = execute(g, inputs, ExecConfig(), ctx=lms_ctx)
    g2, rr = rewrite(g, RewriteConfig(lb=1, ub=3))
    assert rr.tensors_swapped == L
    for codec in ("ce", "sm", "zvc"):
        got, rep = execute(g2, inputs, ExecConfig(codec=codec), ctx=lms_ctx)
        for k in base:
            assert np.array_equal(got[k], base[k]), (codec, k)  # bit-equal
        assert rep.transfer_time_total > 0
        # swapped blocks are held until their D2H lands, so when copies lag the
        # matmuls the peak can exceed no-swap by the tensors still in flight
        assert rep.peak_device_bytes <= rep0.peak_device_bytes + 3 * N * N * 4
    if N <= 256:
        ref = oracle_interpret(g, inputs)
        for k in ref:
            assert _rel(base[k], ref[k]) < 1e-5, k


def test_swapping_fits_a_budget_no_swap_cannot(lms_ctx):
    """Criterion-5 effect on hardware: under a pool limit below the no-swap
    working set, the plain schedule runs out of memory and the rewritten one
    completes with bit-identical results (the pool waits for pending D2H
    copies before refusing an allocation)."""
    L, N = 8, 4096
    tb = N * N * 4
    g = ffchain(L, N)
    inputs = ffchain_inputs(g, N, seed=1)
    execute(g, inputs, ExecConfig(), ctx=lms_ctx)           # warm cuBLAS workspaces
    base, rep0 = execute(g, inputs, ExecConfig(), ctx=lms_ctx)
    g2, _ = rewrite(g, RewriteConfig(lb=1, ub=3))
    torch.cuda.synchronize()
    lms_ctx.synchronize()
    in_use = lms_ctx.stats()["device_in_use"]
    staged = (L + 1) * tb                       # inputs bound by execute()
    limit = in_use + staged + int(0.75 * rep0.peak_device_bytes)
    lms_ctx.set_limit(limit)
    try:
        with pytest.raises(RuntimeError, match="LMS_OOM"):
            execute(g, inputs, ExecConfig(), ctx=lms_ctx)
        torch.cuda.synchronize()
        got, rep = execute(g2, inputs, ExecConfig(codec="ce"), ctx=lms_ctx)
    finally:
        lms_ctx.set_limit(0)
    for k in base:
        assert np.array_equal(got[k], base[k]), k
    assert rep.peak_host_bytes >= L * tb


def test_report_schema(lms_ctx):
    g = ffchain(4, 128)
    g2, _ = rewrite(g, RewriteConfig())
    _, rep = execute(g2, ffchain_inputs(g, 128), ExecConfig(), ctx=lms_ctx)
    d = rep.to_dict()
    assert set(d) == {"peak_device_bytes", "peak_host_bytes", "makespan", "transfer_time_total",
                      "transfer_wait_total", "oom", "event_trace"}
    kinds = {e["event"] for e in d["event_trace"]}
    assert kinds == {"xfer_start", "xfer_finish"}
    assert rep.peak_host_bytes > 0


def test_interpret_dropin_matches_reference_outputs(lms_ctx, interp_cases):
    """``interpret`` keeps the reference signature (interp.py:58) and its float64
    results (golden outputs produced by the reference itself)."""
    from paper_1807_02037_b200 import interpret
    for case in interp_cases:
        inputs = {k: np.asarray(v) for k, v in case["inputs"].items()}
        want = {k: np.asarray(v) for k, v in case["outputs"].items()}
        for rw in case["rewritten"][:1]:
            got = interpret(graph_from_dict(rw["graph"]), inputs, ctx=lms_ctx)
            assert set(got) == set(want)
            for k in want:
                assert np.allclose(got[k], want[k], rtol=1e-12, atol=1e-12), (case["name"], k)
