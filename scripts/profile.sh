#!/bin/bash
# ncu evidence for the staging/transfer kernels (1 GPU).  Outputs under gpurun_out/prof/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
KRE='regex:rows_kernel|transpose_kernel|generic_kernel|copy16_kernel|zvc_'
python scripts/kernel_bench.py ${KB_ARGS:---mib 512} > gpurun_out/prof/kernel_bench.log 2>&1
# launch list of every kernel (ours and the model's) in a short swapped bench step
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-0} -c ${COUNT:-6000} --csv \
  --log-file gpurun_out/prof/launches.csv python bench.py ${PROF_BENCH_ARGS:---steps 1 --warmup 1 --cpu-baseline 0 --b0 193} \
  > gpurun_out/prof/bench_under_ncu.log 2>&1
# full sections for the top kernels of the kernel bench
for k in ${FULL_KERNELS:-zvc_encode_kernel zvc_decode_kernel transpose_kernel copy16_kernel}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof/full_$k python scripts/kernel_bench.py --mib 256 --iters 1 > gpurun_out/prof/full_$k.log 2>&1
done
ls -la gpurun_out/prof
