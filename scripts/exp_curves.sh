#!/bin/bash
# Overhead vs oversubscription (ResNet-50) and the swap-threshold (n_tensors) sweep on ResNet-152 at 3x B0.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 3000 python scripts/overhead_curve.py --b0 193 --factors 1.25,1.5,2,3 > gpurun_out/overhead.log 2>&1; echo "overhead rc=$?"
tail -n 12 gpurun_out/overhead.log
timeout 3000 python scripts/frontier.py --arch resnet152 --factor 3 --lbs 8 --ns 140,200,250,0 > gpurun_out/frontier_thr.log 2>&1; echo "frontier rc=$?"
tail -n 12 gpurun_out/frontier_thr.log
