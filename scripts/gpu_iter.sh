#!/bin/bash
# Iteration pass: GPU tests for the swap engine + kernel bench.  Logs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests} -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python scripts/kernel_bench.py --mib 512 > gpurun_out/kernel_bench.log 2>&1; echo "kb rc=$?"
cat gpurun_out/kernel_bench.log | tail -80
