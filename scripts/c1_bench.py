"""BASELINE configs[0]: the reference's CPU demo path — a feed-forward matmul chain in the
interpreter vocabulary, rewritten with lb=1/ub=3 — run by the GPU executor (execute) vs the
reference executor's semantics on the host (oracle interpret, fp64 numpy, all host threads).

Usage: python scripts/c1_bench.py [--L 8] [--N 1024] [--steps 10]
Prints one JSON object: steps/s on the GPU (fp32, swap on and off, measured SimReport) and on
the CPU (fp64 oracle, swap on), plus the parity checks (swap vs no-swap bit-equal on the GPU;
GPU fp32 vs CPU fp64 relative error).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=8)
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--cpu-steps", type=int, default=3)
    a = ap.parse_args()

    import numpy as np
    import torch
    from oracle.interp_oracle import interpret as oracle_interpret
    from paper_1807_02037_b200 import RewriteConfig, rewrite, runtime as rt
    from paper_1807_02037_b200.executor import ExecConfig, execute
    from paper_1807_02037_b200.workloads import ffchain, ffchain_inputs

    ctx = rt.Context(device=0, device_reserve=8 << 30, timing=True)
    rt.install_allocator(ctx)
    g = ffchain(a.L, a.N)
    inputs = ffchain_inputs(g, a.N, seed=0)
    g2, rep = rewrite(g, RewriteConfig(lb=1, ub=3))
    out = {"workload": f"ffchain L={a.L} N={a.N} (interp vocabulary), RewriteConfig(lb=1, ub=3)",
           "tensors_swapped": rep.tensors_swapped, "control_edges": rep.control_edges_added}
    base, r0 = execute(g, inputs, ExecConfig(), ctx=ctx)
    for label, graph in (("gpu_noswap", g), ("gpu_swap", g2)):
        execute(graph, inputs, ExecConfig(), ctx=ctx)   # warm-up
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(a.steps):
            got, r = execute(graph, inputs, ExecConfig(), ctx=ctx)
        dt = (time.perf_counter() - t) / a.steps
        out[label] = {"steps_per_s": round(1 / dt, 2), "ms_per_step": round(dt * 1e3, 2),
                      "device_makespan_ms": round(r.makespan * 1e3, 3),
                      "peak_device_bytes": r.peak_device_bytes,
                      "transfer_time_total_ms": round(r.transfer_time_total * 1e3, 3),
                      "transfer_wait_total_ms": round(r.transfer_wait_total * 1e3, 3)}
        if label == "gpu_swap":
            out["swap_bit_equal_noswap"] = all(np.array_equal(got[k], base[k]) for k in base)
    threads = len(os.sched_getaffinity(0))
    t = time.perf_counter()
    for _ in range(a.cpu_steps):
        want = oracle_interpret(g2, inputs)
    dt = (time.perf_counter() - t) / a.cpu_steps
    out["cpu_reference_semantics"] = {"steps_per_s": round(1 / dt, 3), "ms_per_step": round(dt * 1e3, 1),
                                      "threads": threads, "dtype": "f64 (interp.py:53-55)"}
    out["gpu_vs_cpu_max_rel_err"] = max(
        float(np.linalg.norm(base[k] - want[k]) / max(np.linalg.norm(want[k]), 1e-300)) for k in want)
    out["note"] = ("wall time per execute() call (host scheduling of ~50 ops included); device_makespan_ms "
                   "is the CUDA-event span of the graph on the compute stream")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
