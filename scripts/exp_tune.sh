#!/bin/bash
# tune_windows: GPU parity test, then the headline and the overhead curve with it on.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/tune
timeout 600 python -m pytest tests/test_torch_swap_gpu.py -x -q > gpurun_out/tune/pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/tune/pytest.log
timeout 900 python bench.py --b0 193 --same-batch 0 --cpu-baseline 0 --tune-windows 1 > gpurun_out/tune/head.json 2> gpurun_out/tune/head.log; echo "head rc=$?"
grep -E "tune_windows|swap batch|OOM|plan:" gpurun_out/tune/head.log | cut -c1-400
timeout 2400 python scripts/overhead_curve.py --b0 193 --factors 1.25,1.5,2,3 --extra="--tune-windows 1" --tag _tuned > gpurun_out/tune/overhead.log 2>&1; echo "overhead rc=$?"
tail -n 9 gpurun_out/tune/overhead.log
