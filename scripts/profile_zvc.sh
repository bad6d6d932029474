#!/bin/bash
# ncu full sections of the ZVC v3 kernels (HBM-side encode/decode, 256 MiB) and a
# DRAM-traffic pass for the zero-copy swap path; summaries land in gpurun_out/.
set -x
cd "$(dirname "$0")/.."
ncu --set full --clock-control none --import-source on -k regex:zvc_encode_kernel -c 2 \
    -o gpurun_out/zvc_encode_full -f python scripts/kernel_bench.py --only zvc --mib 256 --iters 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:zvc_decode_kernel -c 2 \
    -o gpurun_out/zvc_decode_full -f python scripts/kernel_bench.py --only zvc --mib 256 --iters 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:zvc_ --csv --log-file gpurun_out/zvc_swap_traffic.csv python scripts/kernel_bench.py --only swap --mib 256 --iters 2 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/zvc_swap_traffic.csv
