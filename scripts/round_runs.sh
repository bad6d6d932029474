#!/bin/bash
# The round's measured configs (1 GPU): headline bench + reference arm, 3D U-Net, ResNet-152 frontier.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/runs
timeout 1200 python bench.py > gpurun_out/runs/bench.json 2> gpurun_out/runs/bench.log; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/runs/bench_ref.json 2> gpurun_out/runs/bench_ref.log; echo "ref rc=$?"
timeout 1200 python bench.py --arch unet3d --factor 2 --steps 3 > gpurun_out/runs/unet192.json 2> gpurun_out/runs/unet192.log; echo "unet192 rc=$?"
timeout 900 python bench.py --arch unet3d --size 128 --factor 2 --steps 3 --cpu-baseline 0 > gpurun_out/runs/unet128.json 2> gpurun_out/runs/unet128.log; echo "unet128 rc=$?"
timeout 2400 python scripts/frontier.py --arch resnet152 --factor 3 > gpurun_out/runs/frontier.log 2>&1; echo "frontier rc=$?"
cp gpurun_out/frontier_* gpurun_out/runs/ 2>/dev/null
for f in bench bench_ref unet192 unet128; do echo "== $f"; tail -c 600 gpurun_out/runs/$f.json; echo; done
cat gpurun_out/runs/frontier.log | tail -15
