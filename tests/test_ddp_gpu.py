"""Data-parallel replicas with swapping: two ranks, each with its
own liblms pool and swap engine, gradients all-reduced by DDP.

Both ranks share the one GPU of the test box (gloo backend: the all-reduce
goes through the host), so this checks the host-side DP logic — the per-rank
pools, the swapped backward under DDP's bucketed all-reduce hooks, and
``tune_windows`` with its decisions agreed across ranks (every rank takes the
same number of trial steps) — not NVLink bandwidth.  The swapped DDP run must
end with exactly the plain DDP run's parameters on every rank, under a budget
the plain step does not fit in.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "_ddp_worker.py")
GIB = 1 << 30


def _launch(tmp_path, mode, budget):
    env = dict(os.environ, LMS_TEST_NO_POOL="1", CUDNN_CONV_WSCAP_DBG="128", LMS_PAGE_MB="8")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", WORKER, mode, str(tmp_path), f"{budget:.3f}"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    import torch
    return [torch.load(os.path.join(tmp_path, f"{mode}_rank{k}.pt")) for k in range(2)]


def test_swapped_ddp_matches_plain_ddp(tmp_path):
    import torch
    plain = _launch(tmp_path, "plain", 8.0)
    peak = max(p["facts"]["peak"] for p in plain)
    budget = 0.9 * peak / GIB
    swap = _launch(tmp_path, "swap", budget)
    for r in range(2):
        f = swap[r]["facts"]
        assert f["d2h"] > 0 and f["swapped"] > 10
        assert f["tune_restored"]
        assert f["peak"] <= budget * GIB < peak
        for k, v in plain[r]["state"].items():
            assert torch.equal(swap[r]["state"][k], v), (r, k)
    # replicas stay identical (the all-reduce ran on swapped-in activations' gradients)
    for k, v in swap[0]["state"].items():
        if v.is_floating_point() and "running" not in k:
            assert torch.equal(swap[1]["state"][k], v), k
    assert swap[0]["facts"]["tuned"].get("steps_per_trial") == swap[1]["facts"]["tuned"].get("steps_per_trial")


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_one_json_line():
    """bench.py's N>1 contract under torchrun: ranks agree on every fit/tuning
    decision, time with a barrier and take the max over ranks, and rank 0
    alone prints ONE JSON line whose value counts both ranks' images.  (gloo
    lets both ranks share the box's one GPU; --quick, one tuning pass.)"""
    import json
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--quick", "--backend", "gloo", "--cpu-baseline", "0",
           "--tune-windows", "1", "--same-batch", "0"]
    env = dict(os.environ, LMS_BENCH_PG_TIMEOUT_S="180")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2" and d["config"]["pg_backend"] == "gloo"
    bs = d["config"]["per_gpu_batch"]
    assert d["config"]["global_batch"] == 2 * bs
    # whole-job throughput from the max-over-ranks step time
    assert abs(d["value"] - 2 * bs * 1000.0 / d["ms_per_step"]) < 0.01 * d["value"]
    assert d["e2e"]["value"] > 0 and d["swap"]["tensors_swapped"] > 0
    assert isinstance(d["gpu_launches"], int)     # 0 when the codec policy moves every tensor on the copy engine
