"""bench.py's reporting helpers and the auto codec's policy (CPU)."""

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_link_floor():
    import bench
    link = {"d2h": 50.0, "h2d": 40.0, "duplex_total": 80.0}
    f = bench.link_floor(link, 50e9, 40e9, 3000.0, 1200.0)
    assert f["d2h_ms"] == 1000.0 and f["h2d_ms"] == 1000.0 and f["simplex_floor_ms"] == 2000.0
    assert f["duplex_floor_ms"] == pytest.approx(1125.0)   # (50 + 40) GB at 80 GB/s
    assert f["step_over_simplex_floor"] == 1.5 and f["floor_ms"] == pytest.approx(1200.0)
    assert f["step_avg_link_frac"] == pytest.approx(90e9 / 3.0 / 80e9, abs=1e-3)
    assert bench.link_floor({}, 1, 1, 1, None) is None


def test_ncu_traffic_reads_the_committed_capture():
    import bench
    t = bench.ncu_traffic("zvc_encode_kernel")
    d = json.load(open(os.path.join(ROOT, "profiles", "r02", "zvc_swap_traffic.json")))
    assert t["dram_bytes_per_launch"] == round(d["zvc_encode_kernel"]["dram_bytes_per_launch"])
    assert 0.9 < t["ratio"] < 1.1          # the encode reads the tensor once
    assert bench.ncu_traffic("no_such_kernel") is None


def test_zx_policy_follows_link_boundness():
    from paper_1807_02037_b200.torch_lms import SwapExecutor
    p = SwapExecutor.zx_policy
    assert p(0.1, 1.0) == 0.0        # the link has slack: copy engine, no SM kernels
    assert p(0.8, 1.0) == 0.6        # near balance: only clearly compressible tensors
    assert p(1.5, 1.0) == 0.92       # link-bound: every tensor the codec shrinks
    assert p(1.0, 0.0) == 0.92


def test_zx_ratio_estimate_matches_the_codec_rules():
    import torch
    from paper_1807_02037_b200.torch_lms import zx_ratio_estimate
    x = torch.randn(1 << 16)
    assert 0.85 < zx_ratio_estimate(x) < 0.92                    # 4 exponent bits + sign
    assert 0.40 < zx_ratio_estimate(torch.relu(x)) < 0.50        # mask, no sign bit
    assert zx_ratio_estimate(torch.zeros(1 << 16)) < 0.04        # masks only
    assert zx_ratio_estimate(torch.zeros(100)) == 1.0            # under one tile
    assert zx_ratio_estimate(torch.zeros(1 << 16, dtype=torch.float64)) == 1.0   # not 32-bit words
