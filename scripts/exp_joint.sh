#!/bin/bash
# tune_windows=2 (windows + swap-set size): overhead curve and the headline batch.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/joint
timeout 2400 python scripts/overhead_curve.py --b0 193 --factors 1.25,1.5,2,3 --extra="--tune-windows 2" --tag _joint > gpurun_out/joint/overhead.log 2>&1; echo "overhead rc=$?"
tail -n 9 gpurun_out/joint/overhead.log
timeout 1800 python bench.py --b0 193 --same-batch 0 --cpu-baseline 0 --tune-windows 2 > gpurun_out/joint/head.json 2> gpurun_out/joint/head.log; echo "head rc=$?"
grep -E "tune_windows|joint|swap batch|OOM" gpurun_out/joint/head.log | cut -c1-300
