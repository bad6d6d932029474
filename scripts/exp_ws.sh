#!/bin/bash
# Experiment: cuDNN workspace cap vs lb at the headline batch; 3D U-Net 192^3 at a budget where B0 = 1.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/exp
run() { tag=$1; shift; timeout 600 env "$@" > gpurun_out/exp/$tag.json 2> gpurun_out/exp/$tag.log; echo "== $tag rc=$?";
  grep -E "swap batch|OOM at|no-swap|B0=" gpurun_out/exp/$tag.log | tail -4; }
B="python bench.py --b0 193 --same-batch 0 --cpu-baseline 0 --steps 3"
run ws0_lb1 $B --lb 1
run wscap256_lb1 CUDNN_CONV_WSCAP_DBG=256 $B --lb 1
run wscap256_lb2 CUDNN_CONV_WSCAP_DBG=256 $B --lb 2
run wscap256_lb3 CUDNN_CONV_WSCAP_DBG=256 $B --lb 3
run unet_b28 python bench.py --arch unet3d --budget-gib 28 --factor 2 --steps 3 --same-batch 0 --cpu-baseline 0
run unet_b32 python bench.py --arch unet3d --budget-gib 32 --factor 2 --steps 3 --same-batch 0 --cpu-baseline 0
