#!/bin/bash
# ncu evidence for the swap path (1 GPU).  Outputs under gpurun_out/prof/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
python scripts/kernel_bench.py --mib 512 --out gpurun_out/prof/kernel_bench.json > gpurun_out/prof/kernel_bench.log 2>&1
# launch list of every kernel (ours and the model's) in one short swapped bench run
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c ${COUNT:-20000} --csv \
  --log-file gpurun_out/prof/launches.csv python bench.py ${PROF_BENCH_ARGS:---steps 1 --warmup 3 --cpu-baseline 0 --b0 193 --same-batch 0} \
  > gpurun_out/prof/bench_under_ncu.log 2>&1
# full sections: the zero-copy ZVC kernels on the swap path, the HBM staging kernels
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zvc_encode_kernel -s 1 -c 1 \
  -o gpurun_out/prof/full_zvc_encode python scripts/kernel_bench.py --only swap --mib 256 --iters 2 > gpurun_out/prof/full_zvc_encode.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zvc_decode_kernel -s 1 -c 1 \
  -o gpurun_out/prof/full_zvc_decode python scripts/kernel_bench.py --only swap --mib 256 --iters 2 > gpurun_out/prof/full_zvc_decode.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_transpose_kernel -s 2 -c 1 \
  -o gpurun_out/prof/full_tma_transpose python scripts/kernel_bench.py --only pack --mib 256 --iters 1 > gpurun_out/prof/full_tma_transpose.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_copy_kernel -s 2 -c 1 \
  -o gpurun_out/prof/full_tma_pack python scripts/kernel_bench.py --only pack --mib 256 --iters 1 > gpurun_out/prof/full_tma_pack.log 2>&1
ls -la gpurun_out/prof
