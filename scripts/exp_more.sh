#!/bin/bash
# Joint window tuning on the other configs: ResNet-152 at 3x B0 (configs[4]) and 3D U-Net 192^3 at 2x B0 (28 GiB).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/more
timeout 1500 python bench.py --arch resnet152 --factor 3 --b0 90 --same-batch 0 --cpu-baseline 0 --steps 3 > gpurun_out/more/r152.json 2> gpurun_out/more/r152.log; echo "r152 rc=$?"
grep -E "joint|swap batch|OOM" gpurun_out/more/r152.log | cut -c1-200
timeout 1500 python bench.py --arch unet3d --budget-gib 28 --factor 2 --same-batch 0 --cpu-baseline 0 --steps 3 > gpurun_out/more/unet.json 2> gpurun_out/more/unet.log; echo "unet rc=$?"
grep -E "joint|swap batch|OOM|B0" gpurun_out/more/unet.log | cut -c1-200
